// system.h -- the handle behind the opaque ns_system (include/ns.h).
#pragma once
#include <cuda_runtime.h>

#include <vector>

#include "../../include/ns.h"

struct ns_comm;  // comm.cu

namespace ns {
// per-path arrays of the batched kernel (batched.cuh): BLayout.off / in_smem bit order
enum BArr : int { B_X = 0, B_B, B_DX, B_W, B_RI, B_Y, B_VH, B_BE, B_KN, B_NARR };
struct BLayout {
  size_t off[B_NARR];   // doubles, in shared memory (bit set) or in the CTA's global slice
  unsigned in_smem;
  size_t smem_doubles;  // per CTA
  size_t gws_doubles;   // per CTA: A + per-warp series + arrays not in shared memory
  size_t off_A_g;       // A [C][K][d][nnz] in the global slice
  size_t off_ser_g;     // per-warp F/G/X series blocks in the global slice
  int TB;               // diagonal tile of R (power of two <= min(32, n))
};
}  // namespace ns

struct ns_system {
  int dev = 0;
  int n = 0, D = 0, d = 0, K = 0, M = 0, nnz = 0, m_max = 0, max_batch = 1;
  int TB = 32, T = 1;
  int k_lo = 0, dc = 0;
  int n_sample = 0;              // residual sampling (ns_set_residual_sample): 0 = all equations
  int* sample_rows = nullptr;    // [n] device list of the sampled equations  // active stage window [k_lo, dc) of the next step (ns_set_window; default [0, d))
  int sms = 0;
  // host copies
  std::vector<int> h_eq_ptr, h_mono_ptr, h_var_idx, h_row_ptr, h_col_idx, h_mono_dst, h_job_order;
  // device system
  int *eq_ptr = nullptr, *mono_ptr = nullptr, *var_idx = nullptr, *mono_dst = nullptr;
  int *row_ptr = nullptr, *col_idx = nullptr, *job_order = nullptr;
  double *coeff = nullptr, *rhs = nullptr;
  // workspace
  double *b = nullptr, *A = nullptr, *A0 = nullptr, *W = nullptr, *vhead = nullptr, *beta = nullptr;
  double *rdiag = nullptr, *R = nullptr, *Qt = nullptr, *invR = nullptr, *bp = nullptr, *dx = nullptr;
  double *part = nullptr;
  double *Minv = nullptr, *Z = nullptr;  // M = R^{-1} Q^T and its scratch
  bool use_m = true;                  // false: per-stage tiled back substitution (NS_TILED_BS)
  // blocked WY solve (wy.cuh; n > 256 by default, NS_WY overrides): QR of A_0 alone,
  // T_p of BW-reflector blocks, per-stage Q^T b by blocks; V (row-major) lives in Minv
  bool wy = false;
  bool wym = false;            // n <= 256 without the cluster QR: A_0 alone, Q^T = I - V T^T V^T, then M
  double* Vr = nullptr;        // [K][n][n] V row-major (wy / wym)
  int wy_BW = 256, wy_P = 0;
  double *wy_blk = nullptr, *wy_X = nullptr, *wy_T1 = nullptr, *wy_up = nullptr, *wy_u = nullptr;
  int cmax = 1;
  double *y = nullptr, *rbuf = nullptr, *knorm = nullptr, *res_tmp = nullptr, *ws = nullptr;
  int* job_counter = nullptr;
  // eval/diff job queue (evaldiff.cuh): jobs, series pool, progress counters
  int4* jobs = nullptr;
  int njobs = 0, njobs_full = 0;
  int eq_lo = 0, eq_hi = 0;  // equations evaluated by this handle (ns_set_partition)
  long long* ser_off = nullptr;
  double* pool = nullptr;
  int* prog = nullptr;       // [2M]: fprog, gprog
  int* left = nullptr;       // [M]
  int* left_init = nullptr;  // [M]
  long long* trace = nullptr;  // [njobs][3] job trace (NS_TRACE=1 at create), else nullptr
  long long* strace = nullptr; // [d][4] stage-chain stamps (NS_STAGE_TRACE=1 at create), else nullptr
  unsigned* bar = nullptr;     // [4]: qr barrier, stage barrier
  unsigned* status = nullptr;  // device status word
  int grid_ed = 0, grid_qr = 0, grid_st = 0;
  size_t qr_smem_reserve = 0;
  int st_threads = 256;        // threads per CTA of the stage kernel
  int st2_threads = 64, grid_st2 = 0;  // split stage kernel (stage2_kernel): CTA size and grid
  int st2_cwpb = 2;                    // stage2: row-owning warps per critical CTA
  int qr_threads = 128;        // threads per CTA of the QR kernel
  bool qr_owner_beta = false;  // grid QR: the reflector's owner forms beta (NS_QR_OWNER_BETA)
  bool qr_small_regs = false;  // grid QR: register-light variant, 2 CTAs per SM (n > 128)
  bool qr_interleave = true;   // grid QR: column c owned by CTA c mod grid (NS_QR_INTERLEAVE)
  bool qr_crit = false;        // grid QR with a dedicated critical-chain CTA (octo double, n <= 128)
  bool cqr_on = false;         // cluster QR (cqr.cuh) instead of householder_qr_kernel
  int cqr_P = 0, cqr_W = 0, cqr_CPC = 0, cqr_RS = 0, cqr_E = 0;
  size_t cqr_smem = 0;
  bool cqr_withM = false;          // M = R^-1 Q^T formed inside the cluster QR
  long long* cqr_trace = nullptr;  // NS_CQR_TRACE: [n][8] look-ahead stamps (ns_get_qr_trace)
  int conv_terms = 4;          // eval/diff conv: min terms per lane (NS_CONV_TERMS)
  int conv_mode = 0;           // eval/diff conv mode bits (NS_CONV_MODE, evaldiff.cuh)
  bool stage_split = true;     // critical group + right-looking bulk updates (stage2_kernel)
  double* pend = nullptr;      // [K][d][n] pending right-hand sides (stage2)
  double* bpart = nullptr;     // [(d-2) n][K][32] per-lane partial sums of the bulk updates (stage2)
  int* sflags = nullptr;       // [2d + 2] dx published, pend rows done, critical barrier  // dynamic smem requested by the QR kernel to own its SMs
  size_t ed_smem = 0;
  bool qr_cached = false;
  bool no_resid = false;       // this step runs with NS_NO_RESIDUAL
  cudaStream_t last_stream = nullptr;
  // ledger
  static constexpr int LRING = 64;           // pending ledger records (6 events each)
  cudaEvent_t ev[LRING][6] = {};
  // side stream: eval/diff runs there while A_0 -> QR runs on the caller's stream
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  double* A0q = nullptr;
  int* qr_flags = nullptr;  // [n] reflector-ready flags of the QR kernel (epoch valued)
  int qr_epoch = 0;  // dense A_0 as factored (a0_kernel or ns_toeplitz_solve input)
  int ledger_head = 0, ledger_count = 0;     // ring of steps whose events are not yet read
  ns_ledger ledger{};
  int last_launches = 0;
  long long series_products = 0, scale_terms = 0;  // S = sum (3m-5), M + sum m (ledger counts)
  ns_comm* comm = nullptr;     // ns_comm_init (comm.cu), nullptr: one GPU
  // batched (layout, grid and workspace fixed at create: no allocation in a step)
  bool is_complex = false;         // NEXT-2: complex coefficients (batched kernel path)
  bool repeats = false;            // a monomial repeats a variable (exponent > 1, NEXT-3)
  double* bws = nullptr;
  ns::BLayout bl{};
  int b_grid = 0, b_threads = 256, b_minb = 1;
  size_t batched_smem = 0;
  bool btrace_on = false;          // NS_BATCH_TRACE=1 at create: phase stamps of the batched kernel
  long long* strace_b = nullptr;   // [grid][8]
  int btrace_grid = 0;
};


// eval/diff job list of the equations [eq_lo, eq_hi) (api.cu)
void ns_build_jobs(const ns_system* s, int eq_lo, int eq_hi, std::vector<int4>& jobs, std::vector<long long>& ser_off,
                   std::vector<int>& left, long long& pool_series);

// multi-GPU exchange (comm.cu): library-owned NCCL communicator, equation
// partition, row replication of b, A, A_0 after the sharded eval/diff
ns_status ns_comm_exchange(ns_system* s, cudaStream_t st);  // pack own rows, grouped broadcasts, unpack
void ns_comm_free(ns_system* s);
bool ns_comm_active(const ns_system* s);

// per-precision entry points, defined in kernels_k{2,4,8}.cu (impl.cuh)
template <int K>
struct Impl {
  static ns_status setup(ns_system* s);
  static ns_status evaldiff(ns_system* s, const double* x, cudaStream_t st);
  static ns_status qr(ns_system* s, const double* A0src, const double* x, cudaStream_t st);
  static ns_status a0(ns_system* s, const double* x, cudaStream_t st);
  static ns_status stage(ns_system* s, int k_lo, cudaStream_t st);
  static ns_status residual(ns_system* s, double* x, double* res_out, cudaStream_t st);
  static ns_status fabry(ns_system* s, const double* x, double* z, cudaStream_t st);
  static ns_status batched(ns_system* s, int batch, double* x, const double* rhs, double* res,
                           uint32_t flags, cudaStream_t st);
  static ns_status batched_setup(ns_system* s);  // layout, grid, workspace of the batched kernel
  static ns_status md_op(int op, int n, const double* a, const double* b, double* c, cudaStream_t st);
  static ns_status latency(int op, int iters, double* cycles_per_op);
};

#define NS_CK(x)                               \
  do {                                         \
    if ((x) != cudaSuccess) return NS_ECUDA;   \
  } while (0)

template <typename T>
inline cudaError_t ns_dalloc(T** p, size_t count) {
  return cudaMalloc((void**)p, (count > 0 ? count : 1) * sizeof(T));
}
