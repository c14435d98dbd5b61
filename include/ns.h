/* ns.h -- C ABI of libnewtonmd.so: one Newton step on truncated power series
 * in double-double / quad-double / octo-double arithmetic on B200 (sm_100a).
 *
 * Method: arxiv 2301.12659 (J. Verschelde), PAPER.md.  One call performs one
 * iteration of the Newton pseudo-code over all series orders
 * 0..D:
 *   (A(t), b(t)) := evaluate and differentiate f at x(t)
 *   dx(t) := A(t) \ b(t)  -- Householder QR of A_0 once, then for
 *            k = 0..D: b'_k = b_k - sum_{j>=1} A_j dx_{k-j},
 *            y = Q^T b'_k, back substitution R dx_k = y
 *   report ||b(t) - A(t) dx(t)||
 *   x(t) := x(t) + dx(t)
 *
 * Conventions:
 *  - precision = K = number of limbs: 2 (2d), 4 (4d), 8 (8d).  An md number is
 *    an unevaluated sum of K nonoverlapping doubles, most significant first
 *    (P:135-136).  Arrays of md numbers are stored as K LIMB PLANES (structure
 *    of arrays): limb l of element e is at base[l * plane + e].
 *  - dim n, degree D, d = D + 1 coefficients (reading R1: degree 31 = 32
 *    coefficients).
 *  - Layouts:  x, rhs   [K][n][d]     (variable-major series)
 *              b, dx    [K][d][n]     (coefficient-major vectors)
 *              A        [K][d][nnz]   (structural Jacobian, row CSR pattern)
 *              A0       [K][n][n]     (dense leading block, row-major)
 *              residual [K][3]        (||b||, ||b - A dx||, ||dx||: max over
 *                                      k of the vector 1-norm, reading R16)
 *  - Ownership: the caller owns every pointer it passes; device pointers must
 *    be device memory of the handle's device.  The library owns all workspace
 *    (allocated in ns_system_create, freed in ns_system_destroy).  No call
 *    allocates, and no step call synchronises the host; everything is ordered
 *    on the given CUDA stream (cudaStream_t passed as void*; NULL = legacy).
 *  - Errors: argument/shape errors are detected before any launch and
 *    returned; device-side conditions (zero R_jj, non-finite norms) set a
 *    status word read by ns_get_status.  Nothing is printed, nothing throws.
 *  - Threading: one handle per stream; handles are independent.
 */
#ifndef NS_H_
#define NS_H_
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  NS_OK = 0,
  NS_EINVAL = 1,     /* bad argument (NULL pointer, negative size, bad flag)          */
  NS_EPREC = 2,      /* precision not in {2,4,8} or not the handle's precision          */
  NS_EDIM = 3,       /* dim / degree / batch do not match the handle                    */
  NS_EMONO = 4,      /* malformed monomial list (empty, decreasing, >= dim)            */
  NS_ESINGULAR = 5,  /* (status) an R_jj was exactly zero                  */
  NS_ENONFINITE = 6, /* (status) a norm was not finite                                  */
  NS_ENOMEM = 7,     /* device allocation failed at create                              */
  NS_ECUDA = 8,      /* a CUDA runtime call failed                                      */
  NS_ENCCL = 9,      /* reserved: NCCL failure                                          */
  NS_ESTATE = 10     /* NS_REUSE_QR without a cached factorisation                      */
} ns_status;

/* step flags */
#define NS_REUSE_QR 1u    /* skip the QR of A_0, reuse the cached factors     */
#define NS_NO_RESIDUAL 2u /* skip the residual ("can be omitted"): no residual
                             kernel; the returned ||b - A dx|| is 0                         */
#define NS_LEDGER 4u      /* time the kernel classes with CUDA events (T4 classes)         */
#define NS_TILED_BS 8u    /* per stage: y = Q^T b'_k then tiled back substitution (P:659-663,
                             P:124-126); default: dx_k = M b'_k with M = R^{-1} Q^T formed
                             once per factorisation (same algebra, one matvec per stage)  */

#define NS_QR_ONCE 16u    /* ns_run_newton: factor A_0 in the first iteration only, the
                             paper's "the QR decomposition happens only once";
                             default: refactor while stage 0 is active (reading R34)      */
#define NS_NO_STAGGER 32u /* ns_run_newton: all orders 0..D in every iteration           */

typedef struct ns_system ns_system; /* opaque; owns all device workspace */

typedef struct {
  int32_t dim;        /* n                                                        */
  int32_t degree;     /* D (D+1 coefficients)                                     */
  int32_t precision;  /* K in {2,4,8}                                             */
  int32_t n_monomials;/* M                                                        */
  int32_t max_batch;  /* >= 1; paths for ns_newton_series_step_batched            */
  const int32_t* eq_ptr;   /* host [dim+1]: monomials of eq i = [eq_ptr[i], eq_ptr[i+1])  */
  const int32_t* mono_ptr; /* host [M+1]: variables of monomial t = var_idx[mono_ptr[t]..] */
  const int32_t* var_idx;  /* host: nondecreasing per monomial, < dim; a variable listed e
                              times has exponent e (NEXT-3 general exponents)   */
  const double* coeff;     /* host [C][K][M] md coefficient c_t; NULL = all ones          */
  const double* rhs;       /* host [C][K][dim][D+1] right-hand side series r_i(t)         */
  int32_t is_complex;      /* 0: real (C = 1); 1: complex coefficients and series (NEXT-2,
                              P:630-655), C = 2 component planes, real then imaginary:
                              component c, limb l of element e at base[(c K + l) plane + e].
                              A complex handle runs the batched kernel (4M products,
                              complex Householder): ns_newton_series_step (batch 1) and
                              ns_newton_series_step_batched; every other entry point
                              returns NS_EINVAL for it                                   */
} ns_system_desc;

typedef struct {
  uint32_t status_bits;  /* 1 = zero R_jj seen, 2 = non-finite norm                   */
  int32_t qr_cached;     /* 1 if a factorisation is cached for NS_REUSE_QR            */
} ns_step_info;

/* One iteration of ns_run_newton (staggered Newton).  Norms are the
 * leading limbs of the md norms (max over the active k of the vector 1-norm). */
typedef struct {
  int32_t iter;        /* 1-based                                               */
  int32_t k_lo, dc;    /* active stage window [k_lo, dc) of this iteration      */
  int32_t qr;          /* 1 if A_0 was factored in this iteration               */
  double norm_b;       /* ||b||  over k < dc                            */
  double norm_r;       /* ||b - A dx|| over k < dc                      */
  double norm_dx;      /* ||dx||                                        */
  double ms;           /* device time of the iteration's step (CUDA events)     */
} ns_iter_log;

typedef struct {
  int32_t iterations;  /* iterations run (<= max_iter)                          */
  int32_t converged;   /* 1: every stage 0..D retired (reading R34)             */
  int32_t qr_count;    /* factorisations of A_0 performed                       */
  int32_t k_lo;        /* stages retired at exit                                */
} ns_run_info;

/* kernel classes of T4; updates, qhb and bs are fused into one
 * persistent stage kernel and reported together as "stage".  Like the
 * paper's ledger, operation counts accumulate beside the times:
 * the algorithmic md multiply-adds of each class (triangular
 * convolutions + coefficient scalings; (2/3) n^3 for the QR; nnz d(d-1)/2
 * updates + 2 n^2 d for Q^T b + n^2 d / 2 back substitution; nnz d for the
 * residual; over the active window), and the FP64 flops they cost in this
 * library's md arithmetic (static DADD/DMUL/DFMA counts of md.cuh, FMA = 2). */
typedef struct {
  double ms_convolution; /* eval/diff (side stream, concurrent with the QR) */
  double ms_qr;          /* A_0 + Householder QR + tile inverses + M       */
  double ms_stage;       /* updates + Q^T b + back substitution            */
  double ms_residual;    /* residuals + x update + norms                  */
  double ms_total;       /* whole step (start to end, the overlap included) */
  int64_t steps;         /* ledger steps accumulated                     */
  int64_t qr_count;      /* QR factorisations performed                  */
  int64_t md_fma_convolution, md_fma_qr, md_fma_stage, md_fma_residual; /* md multiply-adds */
  double flops_per_md_fma; /* FP64 flops of one md multiply-add (K = 2: 18, 4: 166, 8: 1176) */
  double fp64_flops;       /* sum of the md_fma counts x flops_per_md_fma               */
} ns_ledger;

/* Create a handle for one system on CUDA device cuda_device; validates the
 * descriptor (NS_EMONO / NS_EPREC / NS_EINVAL), uploads it, sizes and
 * allocates all workspace (NS_ENOMEM).  *out is NULL on failure. */
ns_status ns_system_create(const ns_system_desc* desc, int cuda_device, ns_system** out);
void ns_system_destroy(ns_system* sys);

/* One Newton step (see top).  x_series: device [K][dim][degree+1], updated in
 * place.  residual_out: device [K][3] or NULL.  precision/dim/degree must equal
 * the handle's (NS_EPREC / NS_EDIM).  Asynchronous on stream. */
ns_status ns_newton_series_step(ns_system* sys, int precision, int dim, int degree, double* x_series,
                                double* residual_out, uint32_t flags, void* stream);

/* Same step for `batch` independent paths of the same monomial structure
 * (SURVEY 8(e) C5), one CTA per path (batched.cuh).  x_series: device
 * [batch][C][K][dim][degree+1]; rhs: device [batch][C][K][dim][degree+1] or
 * NULL (= the handle's rhs for every path); residual_out: device
 * [batch][K][3] (real md norms) or NULL.  batch <= max_batch; the layout,
 * grid and workspace were sized at create (no allocation here).  flags: 0
 * (the residual is always formed: NS_EINVAL for any flag). */
ns_status ns_newton_series_step_batched(ns_system* sys, int precision, int dim, int degree, int batch,
                                        double* x_series, const double* rhs, double* residual_out,
                                        uint32_t flags, void* stream);

/* Sharded eval/diff: after ns_set_partition(sys, lo, hi) the
 * eval/diff of this handle (ns_eval_diff) computes only the rows [lo, hi) of b,
 * A and A0 (equation-owner sharding; the other rows are left untouched).  The
 * caller replicates the rows across ranks (all-gather over NVLink) and runs
 * ns_newton_series_step_from on every rank.  NS_EINVAL for an empty or
 * out-of-range partition; synchronises the handle's device. */
ns_status ns_set_partition(ns_system* sys, int eq_lo, int eq_hi);
/* Multi-GPU, one large system (north_star "convolution
 * jobs ... followed by an NCCL reduction ... over NVLink").  The library owns
 * the NCCL communicator.  Bootstrap: rank 0 calls ns_nccl_unique_id, the
 * caller broadcasts the 128 bytes (torch.distributed), every rank calls
 * ns_comm_init with its own handle of the same system on its own GPU.  From
 * then on ns_newton_series_step on every rank evaluates and differentiates
 * only the rank's equations (the contiguous ranges of ns_exchange_plan,
 * balanced by convolution cost), replicates the rows of b, A and A_0 of every
 * rank with one grouped ncclBroadcast per rank block (rows are copied, never
 * summed: no ncclSum on limb planes, so every rank's step is bitwise the
 * one-GPU step), and runs the QR, stage loop and residual replicated.  All of
 * it on the step's stream; no host synchronisation.  Collective: every rank
 * must make the same sequence of step calls.  Loads libnccl.so.2 at run time
 * (the copy already in the process, else NS_NCCL_LIB or the loader path);
 * NS_ENCCL if it can not.  ns_comm_init: NS_EINVAL for a bad rank / nranks
 * (nranks <= dim), NS_ESTATE inside a staggered window, NS_ENOMEM, NS_ENCCL;
 * it synchronises the device and blocks until all ranks joined.
 * ns_eval_diff on a sharded handle computes the rank's rows only. */
ns_status ns_nccl_unique_id(void* uid128);
ns_status ns_comm_init(ns_system* sys, int nranks, int rank, const void* uid128);
/* Host only (no device, no handle): for the system of `desc`, the equation
 * ranges eq_bounds[nranks + 1] of the partition ns_comm_init uses, and the
 * size in doubles of each rank's block (block_doubles may be NULL).  Block
 * layout (the row replication contract): [b rows: for l < K, k < d:
 * b[l][k][lo..hi)] [A entries: for l, k: A[l][k][row_ptr[lo]..row_ptr[hi])]
 * [A_0 rows: for l: A_0[l][lo..hi][0..n)]. */
ns_status ns_exchange_plan(const ns_system_desc* desc, int nranks, int32_t* eq_bounds, int64_t* block_doubles);
/* The pack / unpack kernel of the replication (device arrays, layouts as
 * above): unpack = 0 copies rows [lo, hi) of (b, A, A0) into block, unpack = 1
 * copies block into those rows.  Asynchronous on stream. */
ns_status ns_pack_rows(const ns_system* sys, int lo, int hi, double* b, double* A, double* A0, double* block,
                       int unpack, void* stream);
/* NCCL asynchronous error of the handle's communicator (0 = none; NS_ENCCL
 * when set).  NS_OK without a communicator. */
ns_status ns_comm_status(ns_system* sys, int32_t* nccl_async_error);

/* The step after eval/diff: QR of the given A0, stage loop, residual and
 * x += dx, for (b, A, A0) computed elsewhere (all device, layouts as above). */
ns_status ns_newton_series_step_from(ns_system* sys, int precision, int dim, int degree, double* x_series,
                                     const double* b, const double* A, const double* A0,
                                     double* residual_out, uint32_t flags, void* stream);

/* Parity/debug entry points: the same kernels as the step. */
/* eval/diff only: b [K][d][n], A [K][d][nnz], A0 [K][n][n], all device */
ns_status ns_eval_diff(ns_system* sys, const double* x_series, double* b, double* A, double* A0,
                       void* stream);
/* the structural pattern (host arrays [dim+1] and [nnz]); nnz via ns_nnz */
int32_t ns_nnz(const ns_system* sys);
ns_status ns_jacobian_pattern(const ns_system* sys, int32_t* row_ptr, int32_t* col_idx);
/* solve only: QR of A0, then the stage loop for the given b, A; dx [K][d][n] device */
ns_status ns_toeplitz_solve(ns_system* sys, const double* b, const double* A, const double* A0,
                            double* dx, void* stream);
/* R's diagonal (alpha_j, device [K][n]) of the cached factorisation */
ns_status ns_get_r_diag(ns_system* sys, double* rdiag, void* stream);
/* md primitives on device planar arrays [K][n]: op 0 add, 1 mul, 2 fma c+a*b
 * (c input/output), 3 div a/b, 4 sqrt a, 5 sub a-b (tests of row a0) */
ns_status ns_md_op(int precision, int op, int n, const double* a, const double* b, double* c,
                   void* stream);

/* FP64 pipe microbenchmark: op 0 = DFMA chains, 1 = DADD chains on
 * every SM; writes the achieved rate in G instructions/s and the kernel time.
 * Synchronises the device (measurement entry, not part of the step). */
ns_status ns_fp64_peak_probe(int device, int op, double* ginstr_per_s, double* ms);
/* Cost of one grid barrier of the cooperative kernels (microseconds) for a
 * grid of `blocks` x `threads`.  Synchronises. */
ns_status ns_barrier_probe(int device, int blocks, int threads, double* us_per_barrier);
/* Latency of one md operation in a dependent chain on one warp (SM cycles):
 * op 0 fused accumulate, 1 add, 2 mul, 3 reciprocal, 4 sqrt.  Synchronises. */
ns_status ns_md_latency_probe(int precision, int op, double* cycles_per_op);

/* Synchronises the handle's last stream and returns the device status word. */
ns_status ns_get_status(ns_system* sys, ns_step_info* host_out);

/* Active stage window of the following steps (staggered computations,
 * P:494-518): a step evaluates and differentiates at coefficients 0..dc-1
 * only (the products of Eq.(14) truncated at t^dc), solves the stages
 * k = k_lo..dc-1 with dx_k = 0 for the retired stages k < k_lo (Eq.(11):
 * b_k = 0 => dx_k = 0), updates x_k for k < dc only (x_k, k >= dc, are left
 * unchanged) and takes the norms over k < dc.  0 <= k_lo < dc <= degree + 1,
 * else NS_EINVAL.  ns_set_window(sys, 0, degree + 1) restores the full step.
 * Host-side state; stream-ordered with the steps that follow. */
ns_status ns_set_window(ns_system* sys, int k_lo, int dc);

/* Residual sampling (NEXT-4: "select at random one or a couple
 * of equations and compute the residuals for those selected equations"):
 * following steps compute r_k,i = b'_k,i - (A_0 dx_k)_i only for the count
 * distinct equations rows[0..count) (host array, each < dim), and ||r|| is
 * max_k sum over those rows.  count = 0 restores all equations.  NS_EINVAL
 * for a repeated or out-of-range row.  Synchronises the device (upload). */
ns_status ns_set_residual_sample(ns_system* sys, const int32_t* rows, int count);

/* Fabry ratios (NEXT-4; Theorem 1, numerical interpretation
 * P:210-219): z[K][dim] (device) = c_{D-1} / c_D of each series x_j of
 * x_series (device [K][dim][D+1]); |z_j| estimates the radius of convergence.
 * c_D = 0 gives +inf.  NS_EINVAL for degree 0.  Asynchronous on stream. */
ns_status ns_fabry_ratio(ns_system* sys, const double* x_series, double* z, void* stream);

/* Per-stage norms of the last step (synchronises its stream): host_out
 * [4][K][D+1] md values sum_i |v_k,i| for v = b, b - A dx, dx and x (x before
 * the update); entries k >= dc of the last window are stale. */
ns_status ns_get_stage_norms(ns_system* sys, double* host_out);

/* The staggered Newton driver (P:304-325 with P:494-518, SPEC run_newton):
 * x (device [K][dim][D+1], in/out) is the start series, x_0 accurate to about
 * half the working precision.  Iteration i runs one step on the
 * window [k_lo, dc): dc starts at 1 and grows by d := d + 1 + floor(d/2)
 * (Eq.(10)) capped at D+1; after the step stage k_lo retires while
 * ||dx_k|| <= eps ||x_k|| (relative, reading R34; eps <= 0: 1e3 eps_p with
 * eps_p = 2^-104, 2^-210, 2^-423) or ||dx_k|| has reached its rounding floor
 * (<= sqrt(eps_p) ||x_k|| and not below 1/8 of its previous value).  A_0 is factored while stage 0 is active
 * (x_0 still moves) and reused afterwards (x_0 frozen: the cached factors are
 * exact); NS_QR_ONCE factors in iteration 1 only.  Exits when all
 * stages 0..D are retired (converged = 1) or after max_iter iterations.
 * Synchronises the stream once per iteration (the exit test reads the norms).
 * log: host [max_iter] or NULL; info: host or NULL.  flags: NS_QR_ONCE |
 * NS_NO_STAGGER | NS_LEDGER | NS_TILED_BS.  The window is reset to the full
 * step on return. */
ns_status ns_run_newton(ns_system* sys, int precision, int dim, int degree, double* x_series, int max_iter,
                        double eps, uint32_t flags, void* stream, ns_iter_log* log, ns_run_info* info);
/* Job trace of the last eval/diff (handle created with env NS_TRACE=1): per job
 * [pop, inputs ready, done] globaltimer nanoseconds into host[3*i..], the job
 * descriptors {type, monomial/equation, j, key} into jobs_out[4*i..] (may be
 * NULL).  Synchronises.  Returns the number of jobs, -1 without a trace. */
int32_t ns_get_trace(ns_system* sys, int64_t* host, int32_t capacity_jobs, int32_t* jobs_out);
/* Look-ahead trace of the last cluster QR (handle created with env
 * NS_CQR_TRACE=1): per step j, 8 globaltimer stamps (ns) of the warp owning
 * column j+1: [start, reflector rows in, partial dots done, v0 in, beta in,
 * column updated, rows published, reflector j+1 published] into host[8*j..].
 * Synchronises.  Returns the number of steps, -1 without a trace. */
int32_t ns_get_qr_trace(ns_system* sys, int64_t* host, int32_t capacity_steps);
/* Stage-chain trace of the last split stage loop (handle created with env
 * NS_STAGE_TRACE=1): per stage k, 4 globaltimer stamps (ns) of the critical
 * chain: start, pending rhs complete, b'_k written, dx_k written; then [d]
 * stamps of the bulk: the last row of pend_k complete.  host_out holds 5 d
 * values.  Returns d, or -1 without a trace. */
int32_t ns_get_stage_trace(ns_system* sys, int64_t* host_out);
/* Phase trace of the last batched step (handle created with env
 * NS_BATCH_TRACE=1): per CTA, 8 globaltimer stamps (ns) of its first path:
 * start, eval/diff, QR, tile inverses / M, stage loop, residual + update, -, -.
 * Synchronises.  Returns the number of CTAs, -1 without a trace. */
int32_t ns_get_batch_trace(ns_system* sys, int64_t* host, int32_t capacity_ctas);
/* Synchronises; per-class milliseconds accumulated over steps run with NS_LEDGER. */
ns_status ns_get_ledger(ns_system* sys, ns_ledger* host_out);
ns_status ns_reset_ledger(ns_system* sys);
/* Kernels launched by the last step call (for the bench's gpu_launches). */
int32_t ns_last_launch_count(const ns_system* sys);
const char* ns_strerror(ns_status s);
const char* ns_build_info(void);

#ifdef __cplusplus
}
#endif
#endif /* NS_H_ */
