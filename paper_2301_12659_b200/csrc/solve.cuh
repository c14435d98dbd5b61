// solve.cuh -- the linear-algebra half of the Newton step:
//   householder_qr_kernel : Householder QR of A_0, applied to the
//                           augmented [A_0 | I] so that one pass yields R and Q^T
//   invert_tiles_kernel   : inverses of the diagonal tiles of R, once per QR
//                           (tiled back substitution)
//   stage_kernel          : for k = k_lo..D:
//                             b'_k = b_k - sum_{j=1}^{k} A_j dx_{k-j}   (updates)
//                             y    = Q^T b'_k                           (qhb)
//                             R dx_k = y by tiles, last to first        (bs)
//   residual_kernel       : r_k = b'_k - A_0 dx_k (= b_k - sum_{j<=k} A_j dx_{k-j},
//                           reading R17) and the per-k 1-norms of r, b, dx
//   finalize_kernel       : x += dx; ||b||, ||r||, ||dx|| = max_k (reading R16)
// Cooperative kernels use a grid barrier; one warp owns one row or column so
// every md reduction has a fixed order (deterministic).
#pragma once
#include "common.cuh"
#include "evaldiff.cuh"
#include "scalar.cuh"

namespace ns {

__device__ __forceinline__ int gwarp() { return (blockIdx.x * blockDim.x + threadIdx.x) >> 5; }
__device__ __forceinline__ int nwarps() { return (gridDim.x * blockDim.x) >> 5; }
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// warp dot sum_t a_t b_t over t = t0, t0 + dt, ... < t1 (per lane), as
// unnormalised level sums (md::prod_levels + level_insert: no renormalisation
// per term) and one lazy-level butterfly over the warp
template <int K, typename Term>
__device__ __forceinline__ md::mdv<K> warp_dot_levels(int t0, int t1, int dt, Term term) {
  double sl[K];
#pragma unroll
  for (int l = 0; l < K; ++l) sl[l] = 0.0;
  for (int t = t0; t < t1; t += dt) {
    md::mdv<K> a, b;
    term(t, a, b);
    double pl[K];
    md::prod_levels<K>(a, b, pl);
#pragma unroll
    for (int l = 0; l < K; ++l) md::level_insert<K>(sl, l, pl[l]);
  }
  return md::group_sum_levels<K>(sl, 32);
}

// ------------------------------------------------------------------ QR
// W: column-major work matrix, limb planes: W[(l*ncol + c)*n + r], ncol = 2n.
template <int K, bool CG>
MD_INL md::mdv<K> ld(const double* base, long long stride, long long i) {
  return CG ? md::load_cg<K>(base, stride, i) : md::load<K>(base, stride, i);
}
template <int K, bool CG>
MD_INL void st(double* base, long long stride, long long i, const md::mdv<K>& v) {
  if (CG) md::store_cg<K>(base, stride, i, v);
  else md::store<K>(base, stride, i, v);
}

template <int K, bool CG = true>
__device__ void make_reflector(int n, int j, double* W, double* vhead, double* beta, double* rdiag,
                               unsigned* status) {
  const int ncol = 2 * n;
  const long long ls = (long long)ncol * n;
  const int lane = lane_id();
  md::mdv<K> sig = md::zero<K>();
  for (int r = j + lane; r < n; r += 32) {
    md::mdv<K> v = ld<K, CG>(W, ls, (long long)j * n + r);
    sig = md::fma_acc<K>(sig, v, v);
  }
  sig = md::group_sum<K>(sig, 32);
  const md::mdv<K> x0 = ld<K, CG>(W, ls, (long long)j * n + j);
  md::mdv<K> nrm = md::sqrt<K>(sig);
  // alpha = -sign(x0) ||x||, sign(0) = +1 (reading R13)
  md::mdv<K> alpha = md::is_negative<K>(x0) ? nrm : md::neg<K>(nrm);
  md::mdv<K> v0 = md::sub<K>(x0, alpha);
  md::mdv<K> bt = md::zero<K>();
  if (!md::is_zero<K>(sig)) {
    // v^T v = -2 alpha v0, beta = 2 / v^T v = -1 / (alpha v0)
    bt = md::neg<K>(md::recip<K>(md::mul<K>(alpha, v0)));
  } else if (lane == 0 && status) {
    atomicOr(status, ST_SINGULAR);
  }
  if (lane == 0) {
    st<K, CG>(vhead, n, j, v0);
    st<K, CG>(beta, n, j, bt);
    if (rdiag) st<K, CG>(rdiag, n, j, alpha);
    st<K, CG>(W, ls, (long long)j * n + j, alpha);
  }
}

// column c -= beta_j v (v^T column c), rows j..n-1
template <int K, bool CG = true>
__device__ void apply_reflector(int n, int j, int c, double* W, const double* vhead, const double* beta) {
  const int ncol = 2 * n;
  const long long ls = (long long)ncol * n;
  const int lane = lane_id();
  const md::mdv<K> v0 = ld<K, CG>(vhead, n, j);
  md::mdv<K> dot = md::zero<K>();
  for (int r = j + lane; r < n; r += 32) {
    md::mdv<K> v = (r == j) ? v0 : ld<K, CG>(W, ls, (long long)j * n + r);
    md::mdv<K> w = ld<K, CG>(W, ls, (long long)c * n + r);
    dot = md::fma_acc<K>(dot, v, w);
  }
  dot = md::group_sum<K>(dot, 32);
  const md::mdv<K> bt = ld<K, CG>(beta, n, j);
  const md::mdv<K> nw = md::neg<K>(md::mul<K>(bt, dot));
  for (int r = j + lane; r < n; r += 32) {
    md::mdv<K> v = (r == j) ? v0 : ld<K, CG>(W, ls, (long long)j * n + r);
    md::mdv<K> w = ld<K, CG>(W, ls, (long long)c * n + r);
    w = md::fma_acc<K>(w, nw, v);
    st<K, CG>(W, ls, (long long)c * n + r, w);
  }
}

// Reflector jj from sigma = sum_{r >= jj} x_r^2 (already reduced over the
// warp) and x0 = x_jj: alpha = -sign(x0) sqrt(sigma), v0 = x0 - alpha; writes
// vhead = v0, beta slot = alpha v0 (consumers form beta = -1/(alpha v0)), rdiag
// and W[jj][jj] = alpha.
template <int K>
__device__ void reflector_from_sigma(int n, int jj, const md::mdv<K>& sig, const md::mdv<K>& x0, double* W,
                                     double* vhead, double* beta, double* rdiag, unsigned* status,
                                     bool owner_beta = false, long long ls = -1) {
  if (ls < 0) ls = 2LL * n * n;  // W = [A0 | I] (ncol = 2n); the WY path passes n^2
  const int lane = lane_id();
  const md::mdv<K> nrm = md::sqrt<K>(sig);
  const md::mdv<K> alpha = md::is_negative<K>(x0) ? nrm : md::neg<K>(nrm);
  const md::mdv<K> v0 = md::sub<K>(x0, alpha);
  // beta = -1/(alpha v0) is formed by the consumers; store alpha v0 (0 for a zero column)
  md::mdv<K> pav = md::zero<K>();
  if (!md::is_zero<K>(sig)) {
    pav = md::mul<K>(alpha, v0);
    if (owner_beta) pav = md::neg<K>(md::recip<K>(pav));  // the slot holds beta itself
  }
  else if (lane == 0 && status) atomicOr(status, ST_SINGULAR);
  if (lane == 0) {
    md::store_cg<K>(vhead, n, jj, v0);
    md::store_cg<K>(beta, n, jj, pav);
    md::store_cg<K>(rdiag, n, jj, alpha);
    md::store_cg<K>(W, ls, (long long)jj * n + jj, alpha);
  }
}

__device__ __forceinline__ void flag_wait(const int* f, int v) {
  while (ld_relaxed_s32(f) < v) {
  }
  int cur;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(cur) : "l"(f) : "memory");
  (void)cur;
}
// all lanes' prior writes are ordered by the caller's __syncwarp; the release
// store (after an acq_rel fence, cumulative) publishes them
__device__ __forceinline__ void flag_set(int* f, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(f), "r"(v) : "memory");
}

// Householder QR of [A0 | I] (column major, ncol = 2n), one warp per column
// (columns dealt round robin over the co-resident warps).  No grid barrier per
// column: reflector j is published with a release flag; a warp applies H_j to
// its columns once it acquires flag j.  The owner of column j+1 updates that
// column first, keeps it in registers and builds reflector j+1 at once
// (look-ahead of one column), so the critical path is one column update plus
// one reflector per step.  n <= 128 rows per lane-register window (4 x 32).
// SR = rows per lane kept in registers (32 SR rows; the rest streamed from L2):
// SR = 1 (large n, C4) fits 2 CTAs of 256 threads per SM (16 warps: the column
// updates are throughput work and one warp per SMSP left the FP64 pipe idle)
template <int K, int SR = (K == 8) ? 2 : 4>
__global__ void __launch_bounds__(256, (SR == 1) ? 2 : 1) householder_qr_kernel(DevSys sy, const double* __restrict__ x, int n,
                                                             const double* __restrict__ A0,
                                                             double* W, double* vhead, double* beta,
                                                             double* rdiag, unsigned* bar,
                                                             unsigned* status, int* flags, int epoch,
                                                             int owner_beta, int ncol, int interleave) {
  // ncol = 2n: [A0 | I] (R and Q^T in one pass); ncol = n: A0 alone (WY path, wy.cuh)
  const long long ls = (long long)ncol * n;
  const int gw = gwarp(), nw = nwarps(), lane = lane_id();
  // W = [A0 | I], column major.  With x given, A_0 is formed here (warp per
  // equation, a0_row) so the QR needs no eval/diff output and can start first.
  const long long tot = (long long)K * ncol * n;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < tot;
       t += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(t % n);
    const long long lc = t / n;
    const int c = (int)(lc % ncol), l = (int)(lc / ncol);
    if (c < n && x) continue;
    double v;
    if (c < n) v = A0[((long long)l * n + r) * n + c];
    else v = (l == 0 && r == c - n) ? 1.0 : 0.0;
    __stcg(W + (long long)l * ls + (long long)c * n + r, v);
  }
  if (x)
    for (int i = gw; i < n; i += nw) a0_row<K>(sy, x, i, W, ls, 1, n);
  {
    GridBarrier gb(bar, (unsigned)(epoch - 1) * (gridDim.x * gridDim.y * gridDim.z));
    gb.sync();
  }
  // column ownership: warp w of CTA b owns columns ow, ow + nw, ... with
  // ow = w G + b (interleave = 1): every SM holds columns spread over the whole
  // range, so the SMs stay busy until the end (with ow = global warp id, CTA b
  // owned columns 8b..8b+7 and the SMs of the early columns idled: half the
  // GPU for the second half of the factorisation)
  const int ow = interleave ? (int)((threadIdx.x >> 5) * gridDim.x + blockIdx.x) : gw;
  if (ow == 0) {  // reflector 0 (owner of column 0)
    md::mdv<K> sig = md::zero<K>();
    for (int r = lane; r < n; r += 32) {
      const md::mdv<K> v = md::load_cg<K>(W, ls, r);
      sig = md::fma_acc<K>(sig, v, v);
    }
    sig = md::group_sum<K>(sig, 32);
    reflector_from_sigma<K>(n, 0, sig, md::load_cg<K>(W, ls, 0), W, vhead, beta, rdiag, status, owner_beta != 0, ls);
    __syncwarp();
    if (lane == 0) flag_set(flags + n, epoch);  // B[0]
  }
  // Two flags per column j (epoch valued): A[j] = column j final below the
  // diagonal (rows > j), B[j] = reflector j (vhead, beta) published.  After A[j]
  // every warp forms the partial dot sum_{r>j} v_r W[r][c] of its columns while
  // the owner of column j is still computing the norm, sqrt and reciprocal;
  // after B[j] it adds v0 W[j][c] and applies the update.
  int* fA = flags;
  int* fB = flags + n;
  constexpr int S = SR;  // rows per lane kept in registers (32 S rows)
  for (int j = 0; j < n; ++j) {
    // first owned column > j (the look-ahead column j+1 is always its owner's first)
    int c0 = ow;
    if (c0 <= j) c0 += ((j - ow) / nw + 1) * nw;
    if (c0 >= ncol) break;  // nothing left for this warp
    if (j > 0) flag_wait(fA + j, epoch);  // column 0 was final at the start
    __syncwarp();
    // v rows (r > j) and the first column's rows (r >= j) in registers: slot s holds
    // row j + lane + 32 s; rows beyond 32 S are streamed from L2
    md::mdv<K> vr[S], wr[S];
#pragma unroll
    for (int q = 0; q < S; ++q) {
      const int r = j + lane + 32 * q;
      vr[q] = (r > j && r < n) ? md::load_cg<K>(W, ls, (long long)j * n + r) : md::zero<K>();
      wr[q] = (r < n) ? md::load_cg<K>(W, ls, (long long)c0 * n + r) : md::zero<K>();
    }
    constexpr int MAXC = 4;  // partial dots kept in flight per warp (more columns: dot recomputed)
    md::mdv<K> part[MAXC];
    // partial dots as unnormalised level sums, one lazy-level butterfly each
    auto lv_add = [&](double (&sl)[K], const md::mdv<K>& a, const md::mdv<K>& b) {
      double pl[K];
      md::prod_levels<K>(a, b, pl);
#pragma unroll
      for (int l = 0; l < K; ++l) md::level_insert<K>(sl, l, pl[l]);
    };
    {
      double sl[K];
#pragma unroll
      for (int l = 0; l < K; ++l) sl[l] = 0.0;
#pragma unroll
      for (int q = 0; q < S; ++q) {
        const int r = j + lane + 32 * q;
        if (r > j && r < n) lv_add(sl, vr[q], wr[q]);
      }
      for (int r = j + lane + 32 * S; r < n; r += 32)
        lv_add(sl, md::load_cg<K>(W, ls, (long long)j * n + r), md::load_cg<K>(W, ls, (long long)c0 * n + r));
      part[0] = md::group_sum_levels<K>(sl, 32);
    }
    int nc = 1;
    for (int c = c0 + nw; c < ncol && nc < MAXC; c += nw, ++nc) {
      double sl[K];
#pragma unroll
      for (int l = 0; l < K; ++l) sl[l] = 0.0;
      for (int r = j + 1 + lane; r < n; r += 32)
        lv_add(sl, md::load_cg<K>(W, ls, (long long)j * n + r), md::load_cg<K>(W, ls, (long long)c * n + r));
      part[nc] = md::group_sum_levels<K>(sl, 32);
    }
    flag_wait(fB + j, epoch);
    __syncwarp();
    const md::mdv<K> v0 = md::load_cg<K>(vhead, n, j);
    const md::mdv<K> pav = md::load_cg<K>(beta, n, j);  // alpha_j v0_j
    // beta_j = -1 / (alpha v0), formed here (each consumer) so that the owner's
    // critical chain ends at alpha v0; zero column -> beta = 0 (H = I)
    // owner_beta: the owner formed beta once (one reciprocal per reflector instead of one
    // per consumer warp competing for the FP64 pipes); else each consumer forms it
    const md::mdv<K> bt = owner_beta ? pav : (md::is_zero<K>(pav) ? md::zero<K>() : md::neg<K>(md::recip<K>(pav)));
    int ic = 0;
    for (int c = c0; c < ncol; c += nw, ++ic) {
      md::mdv<K> dot;
      if (ic < MAXC) {
        dot = part[ic];
      } else {  // more columns than kept in flight: full dot here
        md::mdv<K> p = md::zero<K>();
        for (int r = j + 1 + lane; r < n; r += 32)
          p = md::fma_acc<K>(p, md::load_cg<K>(W, ls, (long long)j * n + r), md::load_cg<K>(W, ls, (long long)c * n + r));
        dot = md::group_sum<K>(p, 32);
      }
      const bool first = (ic == 0);
      const md::mdv<K> wj = first ? md::shfl<K>(wr[0], 0) : md::load_cg<K>(W, ls, (long long)c * n + j);
      dot = md::fma_acc<K>(dot, v0, wj);
      const md::mdv<K> nw_ = md::neg<K>(md::mul<K>(bt, dot));
      const bool look = (c == j + 1 && c < n);
      // look-ahead norm as unnormalised level sums (no renormalisation per term),
      // one lazy-level butterfly (as in cqr.cuh): a shorter chain to reflector j+1
      double sg[K];
#pragma unroll
      for (int l = 0; l < K; ++l) sg[l] = 0.0;
      md::mdv<K> x0 = md::zero<K>();
      auto sg_add = [&](const md::mdv<K>& w) {
        double pl[K];
        md::prod_levels<K>(w, w, pl);
#pragma unroll
        for (int l = 0; l < K; ++l) md::level_insert<K>(sg, l, pl[l]);
      };
      if (first) {
#pragma unroll
        for (int q = 0; q < S; ++q) {
          const int r = j + lane + 32 * q;
          if (r < n) {
            const md::mdv<K> v = (r == j) ? v0 : vr[q];
            const md::mdv<K> w = md::fma_acc<K>(wr[q], nw_, v);
            md::store_cg<K>(W, ls, (long long)c * n + r, w);
            if (look && r > j) sg_add(w);  // look-ahead norm, same pass
            if (r == j + 1) x0 = w;
          }
        }
        for (int r = j + lane + 32 * S; r < n; r += 32) {
          const md::mdv<K> w =
              md::fma_acc<K>(md::load_cg<K>(W, ls, (long long)c * n + r), nw_, md::load_cg<K>(W, ls, (long long)j * n + r));
          md::store_cg<K>(W, ls, (long long)c * n + r, w);
          if (look) sg_add(w);
        }
      } else {
        for (int r = j + lane; r < n; r += 32) {
          const md::mdv<K> v = (r == j) ? v0 : md::load_cg<K>(W, ls, (long long)j * n + r);
          const md::mdv<K> w = md::fma_acc<K>(md::load_cg<K>(W, ls, (long long)c * n + r), nw_, v);
          md::store_cg<K>(W, ls, (long long)c * n + r, w);
        }
      }
      if (look) {
        __syncwarp();
        if (lane == 0) flag_set(fA + j + 1, epoch);  // column j+1 final below its diagonal
        const md::mdv<K> sig = md::group_sum_levels<K>(sg, 32);
        x0 = md::shfl<K>(x0, 1);  // row j+1 lives in lane 1
        reflector_from_sigma<K>(n, j + 1, sig, x0, W, vhead, beta, rdiag, status, owner_beta != 0, ls);
        __syncwarp();
        if (lane == 0) flag_set(fB + j + 1, epoch);
      }
    }
  }
}

// CTA-wide sum of unnormalised level sums (one per thread): warp butterflies,
// then warp 0 combines the warps' levels in warp order; every thread gets the
// renormalised value.  scratch: K * (blockDim / 32) doubles of shared memory.
template <int K>
__device__ md::mdv<K> block_sum_levels(double (&sl)[K], double* scratch) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double s[K];
#pragma unroll
  for (int l = 0; l < K; ++l) s[l] = sl[l];
  lv_group<K>(s, 32);
  if (lane == 0)
#pragma unroll
    for (int l = 0; l < K; ++l) scratch[w * K + l] = s[l];
  __syncthreads();
  if (w == 0) {
    double t[K];
#pragma unroll
    for (int l = 0; l < K; ++l) t[l] = (lane < nw) ? scratch[lane * K + l] : 0.0;
    lv_group<K>(t, 32);
    const md::mdv<K> v = md::renorm<K, K>(t);
    if (lane == 0)
#pragma unroll
      for (int l = 0; l < K; ++l) scratch[nw * K + l] = v.x[l];
  }
  __syncthreads();
  md::mdv<K> r;
#pragma unroll
  for (int l = 0; l < K; ++l) r.x[l] = scratch[nw * K + l];
  __syncthreads();  // scratch reusable
  return r;
}

// Householder QR of [A0 | I] (or A0 alone) with a dedicated critical CTA.  In the grid QR
// the look-ahead column's owner warp shares its SM's FP64 pipes with seven
// warps doing throughput updates, so the dependent chain (update column j+1,
// its norm, sqrt, reciprocal) ran at a fraction of the pipe: 54 us per step at
// C3.  Here CTA 0 does only that chain, with all its threads on the column:
//   step j: wait U[j+1] (column j+1 has H_0..H_{j-2}), apply H_{j-1} and H_j
//   to it (rows spread over the CTA, CTA-wide dots), publish A[j+1] (rows > j+1
//   final), CTA-wide norm, reflector j+1, publish B[j+1].
// CTAs 1.. own every other column update: column c (c >= 1, dealt round robin
// over their warps) takes H_0..H_{c-3} from its owner warp, which publishes
// U[c] after H_{c-3}; H_{c-2} and H_{c-1} are the critical CTA's (look-ahead of
// two: with one, the owner warp's update of the next column by H_{c-2} sat on
// the chain).  Same arithmetic per
// element as householder_qr_kernel (so the same results up to the order of
// the dot's partial sums).  Flags (epoch valued): A [n], B [n], U [n].
template <int K>
__global__ void __launch_bounds__(256, 1) householder_qr_crit_kernel(DevSys sy, const double* __restrict__ x, int n,
                                                                    const double* __restrict__ A0, double* W,
                                                                    double* vhead, double* beta, double* rdiag,
                                                                    unsigned* bar, unsigned* status, int* flags,
                                                                    int epoch, int ncol, int interleave) {
  __shared__ double scratch[K * 9];
  __shared__ double sx0[K];
  // ncol = 2n: [A0 | I]; ncol = n: A0 alone (WY path)
  const long long ls = (long long)ncol * n;
  const int gw = gwarp(), nw = nwarps(), lane = lane_id();
  const long long tot = (long long)K * ncol * n;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < tot;
       t += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(t % n);
    const long long lc = t / n;
    const int c = (int)(lc % ncol), l = (int)(lc / ncol);
    if (c < n && x) continue;
    double v;
    if (c < n) v = A0[((long long)l * n + r) * n + c];
    else v = (l == 0 && r == c - n) ? 1.0 : 0.0;
    __stcg(W + (long long)l * ls + (long long)c * n + r, v);
  }
  if (x)
    for (int i = gw; i < n; i += nw) a0_row<K>(sy, x, i, W, ls, 1, n);
  {
    GridBarrier gb(bar, (unsigned)(epoch - 1) * (gridDim.x * gridDim.y * gridDim.z));
    gb.sync();
  }
  int* fA = flags;
  int* fB = flags + n;
  int* fU = flags + 2 * n;
  if (blockIdx.x == 0) {
    // ---------------- the critical chain
    const int NT = blockDim.x;
    {  // reflector 0
      double sl[K];
      lv_zero<K>(sl);
      for (int r = threadIdx.x; r < n; r += NT) {
        const md::mdv<K> v = md::load_cg<K>(W, ls, r);
        lv_prod<K>(sl, v, v);
      }
      const md::mdv<K> sig = block_sum_levels<K>(sl, scratch);
      if (threadIdx.x < 32) {
        reflector_from_sigma<K>(n, 0, sig, md::load_cg<K>(W, ls, 0), W, vhead, beta, rdiag, status, true, ls);
        __syncwarp();
        if (lane == 0) flag_set(fB, epoch);
      }
      __syncthreads();
    }
    for (int j = 0; j + 1 < n; ++j) {
      const int c = j + 1;
      // column c arrives with H_0..H_{c-3} from its owner warp (U[c]); this CTA
      // applies H_{c-2} = H_{j-1} and H_{c-1} = H_j itself (look-ahead of two:
      // the owner warp's update of a full column is not on the chain)
      if (j >= 2) {
        if (threadIdx.x == 0) flag_wait(fU + c, epoch);
        __syncthreads();
      }
      double sg[K];
      lv_zero<K>(sg);
      for (int jj = (j >= 1 ? j - 1 : j); jj <= j; ++jj) {
        const md::mdv<K> v0 = md::load_cg<K>(vhead, n, jj);
        const md::mdv<K> bt = md::load_cg<K>(beta, n, jj);  // beta itself (the owner forms it)
        double sl[K];
        lv_zero<K>(sl);
        for (int r = jj + threadIdx.x; r < n; r += NT) {
          const md::mdv<K> v = (r == jj) ? v0 : md::load_cg<K>(W, ls, (long long)jj * n + r);
          lv_prod<K>(sl, v, md::load_cg<K>(W, ls, (long long)c * n + r));
        }
        const md::mdv<K> dot = block_sum_levels<K>(sl, scratch);
        const md::mdv<K> nw_ = md::neg<K>(md::mul<K>(bt, dot));
        const bool last = (jj == j);
        for (int r = jj + threadIdx.x; r < n; r += NT) {
          const md::mdv<K> v = (r == jj) ? v0 : md::load_cg<K>(W, ls, (long long)jj * n + r);
          const md::mdv<K> w = md::fma_acc<K>(md::load_cg<K>(W, ls, (long long)c * n + r), nw_, v);
          md::store_cg<K>(W, ls, (long long)c * n + r, w);
          if (last && r >= c) lv_prod<K>(sg, w, w);  // sigma = sum_{r >= c} x_r^2
          if (last && r == c) md::store<K>(sx0, 1, 0, w);
        }
        __syncthreads();  // the column's rows, written by other threads, feed the next dot
      }
      if (threadIdx.x == 0) flag_set(fA + c, epoch);  // rows > c final (cumulative after the barrier)
      const md::mdv<K> sig = block_sum_levels<K>(sg, scratch);
      if (threadIdx.x < 32) {
        reflector_from_sigma<K>(n, c, sig, md::load<K>(sx0, 1, 0), W, vhead, beta, rdiag, status, true, ls);
        __syncwarp();
        if (lane == 0) flag_set(fB + c, epoch);
      }
      __syncthreads();
    }
    return;
  }
  // ---------------- the column updates: warps of CTAs 1.., column c (c >= 1)
  // interleave: warp w of CTA b (b >= 1) owns columns 1 + w (G - 1) + (b - 1), ... (every SM
  // holds columns spread over the whole range, as in householder_qr_kernel)
  const int rw = interleave ? (int)((threadIdx.x >> 5) * (gridDim.x - 1) + blockIdx.x - 1)
                            : (int)((blockIdx.x - 1) * (blockDim.x >> 5) + (threadIdx.x >> 5));
  const int nrw = (gridDim.x - 1) * (blockDim.x >> 5);
  for (int j = 0; j + 1 < ncol && j < n; ++j) {
    // owned columns c > j, except the chain columns c in {j+1, j+2} (c < n: H_{c-2}
    // and H_{c-1} are the critical CTA's); the columns of I (c >= n) take every H_j
    int c0 = 1 + rw;
    if (c0 <= j) c0 += ((j - c0) / nrw + 1) * nrw;
    if (c0 >= ncol) break;
    auto chain_col = [&](int cc) { return cc < n && cc <= j + 2; };
    if (j > 0) flag_wait(fA + j, epoch);
    __syncwarp();
    constexpr int MAXC = 4;
    md::mdv<K> part[MAXC];
    int nc = 0;
    for (int cc = c0; cc < ncol && nc < MAXC; cc += nrw) {  // partial dots over rows > j
      if (chain_col(cc)) continue;
      double sl[K];
      lv_zero<K>(sl);
      for (int r = j + 1 + lane; r < n; r += 32)
        lv_prod<K>(sl, md::load_cg<K>(W, ls, (long long)j * n + r), md::load_cg<K>(W, ls, (long long)cc * n + r));
      part[nc++] = md::group_sum_levels<K>(sl, 32);
    }
    flag_wait(fB + j, epoch);
    __syncwarp();
    const md::mdv<K> v0 = md::load_cg<K>(vhead, n, j);
    const md::mdv<K> bt = md::load_cg<K>(beta, n, j);
    int ic = 0;
    for (int cc = c0; cc < ncol; cc += nrw) {
      if (chain_col(cc)) continue;
      md::mdv<K> dot;
      if (ic < MAXC) {
        dot = part[ic];
      } else {
        double sl[K];
        lv_zero<K>(sl);
        for (int r = j + 1 + lane; r < n; r += 32)
          lv_prod<K>(sl, md::load_cg<K>(W, ls, (long long)j * n + r), md::load_cg<K>(W, ls, (long long)cc * n + r));
        dot = md::group_sum_levels<K>(sl, 32);
      }
      ++ic;
      dot = md::fma_acc<K>(dot, v0, md::load_cg<K>(W, ls, (long long)cc * n + j));
      const md::mdv<K> nw_ = md::neg<K>(md::mul<K>(bt, dot));
      constexpr int QB = (K == 8) ? 2 : 4;  // rows per lane loaded together
      for (int rb = j + lane; rb < n; rb += 32 * QB) {
        md::mdv<K> wq[QB], vq[QB];
#pragma unroll
        for (int q = 0; q < QB; ++q) {
          const int r = rb + 32 * q;
          if (r < n) {
            wq[q] = md::load_cg<K>(W, ls, (long long)cc * n + r);
            vq[q] = (r == j) ? v0 : md::load_cg<K>(W, ls, (long long)j * n + r);
          }
        }
#pragma unroll
        for (int q = 0; q < QB; ++q) {
          const int r = rb + 32 * q;
          if (r < n) md::store_cg<K>(W, ls, (long long)cc * n + r, md::fma_acc<K>(wq[q], nw_, vq[q]));
        }
      }
      if (cc == j + 3 && cc < n) {  // H_0..H_{cc-3} applied: the critical CTA may take it
        __syncwarp();
        if (lane == 0) flag_set(fU + cc, epoch);
      }
    }
  }
}

// Row-major copies for the stage loop: R[r][c] (upper, diagonal = alpha) and
// Qt[r][c] = (Q^T)[r][c].
template <int K>
__global__ void qr_unpack_kernel(int n, const double* __restrict__ W, double* R, double* Qt) {
  const int ncol = 2 * n;
  const long long ls = (long long)ncol * n;
  const long long tot = (long long)K * n * n;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < tot;
       t += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(t % n);
    const long long lr = t / n;
    const int r = (int)(lr % n), l = (int)(lr / n);
    R[t] = (c >= r) ? W[l * ls + (long long)c * n + r] : 0.0;
    Qt[t] = W[l * ls + (long long)(n + c) * n + r];
  }
}

// Inverse of the diagonal tile t of R (size nb <= TB = 32) by recursive
// doubling: inv([[A, B], [0, C]]) = [[inv A, -inv A B inv C], [0, inv C]],
// levels s = 2, 4, ..., 32; each level is two small products whose entries
// are independent (one thread each), so the dependent chain is
// 2 (1 + 2 + 4 + 8 + 16) = 62 md multiply-adds instead of 32 x (dot + butterfly).
// Rows/columns >= nb are padded with the identity.  invR: [K][T][TB][TB] row-major.
template <int K>
__global__ void __launch_bounds__(256) invert_tiles_kernel(int n, int TB, const double* __restrict__ R,
                                                           double* invR) {
  extern __shared__ double sm[];
  const int t = blockIdx.x;
  const int t0 = t * TB;
  const int nb = min(TB, n - t0);
  const int T = (n + TB - 1) / TB;
  const long long lsR = (long long)n * n;
  const long long lsI = (long long)T * TB * TB;
  const int TT = TB * TB;
  double* sR = sm;                 // [K][TB][TB]
  double* sX = sm + (long long)K * TT;  // [K][TB][TB]
  double* sT = sX + (long long)K * TT;  // [K][TT/2] level scratch
  for (int e = threadIdx.x; e < TT; e += blockDim.x) {
    const int r = e / TB, c = e % TB;
    md::mdv<K> v = md::zero<K>();
    if (r < nb && c < nb) {
      if (c >= r) v = md::load<K>(R, lsR, (long long)(t0 + r) * n + t0 + c);
    } else if (r == c) {
      v = md::from_double<K>(1.0);
    }
    md::store<K>(sR, TT, e, v);
    md::store<K>(sX, TT, e, md::zero<K>());
  }
  __syncthreads();
  for (int r = threadIdx.x; r < TB; r += blockDim.x)
    md::store<K>(sX, TT, r * TB + r, md::recip<K>(md::load<K>(sR, TT, r * TB + r)));
  __syncthreads();
  for (int sz = 2; sz <= TB; sz <<= 1) {
    const int h = sz >> 1;
    const int nent = (TB / sz) * h * h;
    // T1[blk][p][q] = sum_{u=0}^{q} R[base+p][base+h+u] X[base+h+u][base+h+q]
    for (int e = threadIdx.x; e < nent; e += blockDim.x) {
      const int blk = e / (h * h), p = (e / h) % h, q = e % h;
      const int base = blk * sz;
      md::mdv<K> acc = md::zero<K>();
      for (int u = 0; u <= q; ++u)
        acc = md::fma_acc<K>(acc, md::load<K>(sR, TT, (base + p) * TB + base + h + u),
                             md::load<K>(sX, TT, (base + h + u) * TB + base + h + q));
      md::store<K>(sT, TT / 2, e, acc);
    }
    __syncthreads();
    // X[base+p][base+h+q] = - sum_{v=p}^{h-1} X[base+p][base+v] T1[blk][v][q]
    for (int e = threadIdx.x; e < nent; e += blockDim.x) {
      const int blk = e / (h * h), p = (e / h) % h, q = e % h;
      const int base = blk * sz;
      md::mdv<K> acc = md::zero<K>();
      for (int v = p; v < h; ++v)
        acc = md::fma_acc<K>(acc, md::load<K>(sX, TT, (base + p) * TB + base + v),
                             md::load<K>(sT, TT / 2, blk * h * h + v * h + q));
      md::store<K>(sX, TT, (base + p) * TB + base + h + q, md::neg<K>(acc));
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < TT; e += blockDim.x) {
    const int r = e / TB, c = e % TB;
    md::mdv<K> v = (r < nb && c < nb) ? md::load<K>(sX, TT, e) : md::zero<K>();
    md::store<K>(invR, lsI, (long long)t * TT + e, v);
  }
}

// M = R^{-1} Q^T (row-major [K][n][n]) by tiled back substitution on the n
// columns of Q^T, tiles last to first:  Z_t = Q^T_t - sum_{c >= t1} R[t][c] M[c],
// M_t = invR_t Z_t.  Each output entry (r, j) is a dot shared by a group of
// FM_G lanes (lane s of the group sums c = c0 + s, c0 + s + FM_G, ... in
// order, then a fixed butterfly): one lane per entry left every warp with a
// serial chain of up to n 8d multiply-adds (issue bound, 0.92 ms at C3).
// With M each stage's "Q^T b then back substitution" is one matvec
// dx_k = M b'_k (same algebra, R^{-1}(Q^T b) = (R^{-1} Q^T) b).
constexpr int FM_G = 8;
template <int K>
__global__ void __launch_bounds__(256) form_m_kernel(int n, int TB, const double* __restrict__ R,
                                                     const double* __restrict__ Qt, const double* __restrict__ invR,
                                                     double* M, double* Z, unsigned* bar) {
  GridBarrier gb(bar, 0u);
  const int gw = gwarp(), nw = nwarps(), lane = lane_id();
  const int T = (n + TB - 1) / TB;
  const long long lsM = (long long)n * n, lsI = (long long)T * TB * TB;
  constexpr int OPW = 32 / FM_G;  // outputs per warp task
  const int sub = lane % FM_G;
  for (int t = T - 1; t >= 0; --t) {
    const int t0 = t * TB, t1 = min(n, t0 + TB);
    const int nout = (t1 - t0) * n;
    const int tasks = (nout + OPW - 1) / OPW;
    for (int w = gw; w < tasks; w += nw) {
      const int o = w * OPW + lane / FM_G;
      const bool ok = o < nout;
      const int r = ok ? t0 + o / n : t0, j = ok ? o % n : 0;
      double sl[K];
#pragma unroll
      for (int l = 0; l < K; ++l) sl[l] = 0.0;
      if (ok)
        for (int c = t1 + sub; c < n; c += FM_G) {
          double pl[K];
          md::prod_levels<K>(md::load<K>(R, lsM, (long long)r * n + c), md::load_cg<K>(M, lsM, (long long)c * n + j), pl);
#pragma unroll
          for (int l = 0; l < K; ++l) md::level_insert<K>(sl, l, pl[l]);
        }
      const md::mdv<K> acc = md::group_sum_levels<K>(sl, FM_G);
      if (ok && sub == 0)
        md::store_cg<K>(Z, lsM, (long long)r * n + j, md::sub<K>(md::load<K>(Qt, lsM, (long long)r * n + j), acc));
    }
    gb.sync();
    for (int w = gw; w < tasks; w += nw) {
      const int o = w * OPW + lane / FM_G;
      const bool ok = o < nout;
      const int r = ok ? t0 + o / n : t0, j = ok ? o % n : 0;
      double sl[K];
#pragma unroll
      for (int l = 0; l < K; ++l) sl[l] = 0.0;
      if (ok)
        for (int c = t0 + sub; c < t1; c += FM_G) {
          double pl[K];
          md::prod_levels<K>(md::load<K>(invR, lsI, (long long)t * TB * TB + (long long)(r - t0) * TB + (c - t0)),
                             md::load_cg<K>(Z, lsM, (long long)c * n + j), pl);
#pragma unroll
          for (int l = 0; l < K; ++l) md::level_insert<K>(sl, l, pl[l]);
        }
      const md::mdv<K> acc = md::group_sum_levels<K>(sl, FM_G);
      if (ok && sub == 0) md::store_cg<K>(M, lsM, (long long)r * n + j, acc);
    }
    gb.sync();
  }
}

// ------------------------------------------------------------------ stage loop
struct StageArgs {
  const double* b;     // [K][d][n]
  const double* A;     // [K][d][nnz]
  const double* Qt;    // [K][n][n] row-major
  const double* R;     // [K][n][n] row-major upper
  const double* invR;  // [K][T][TB][TB]
  double* bp;          // [K][d][n]  b'_k
  double* dx;          // [K][d][n]
  double* y;           // [K][n]
  double* part;        // [K][n][cmax] partial sums of the update chunks
  const double* M;     // [K][n][n] = R^{-1} Q^T, or nullptr for the per-stage tiled path
  int cmax;            // max chunks per row = ceil((d-1) * maxlen / UCH)
  int TB;
  int k_lo;
};

constexpr int UCH = 64;  // update terms per chunk (32 lanes x 2)

// ---- updates: b'_k = b_k - sum_{j=1}^{k} A_j dx_{k-j}, all warps of a
// cooperative grid.  The k*len_i terms of row i are cut into chunks of UCH;
// (row, chunk) slots are dealt to all warps, each chunk is summed by one warp
// (fixed lane order + butterfly), then the chunks of a row are summed in chunk
// order: deterministic and balanced whatever the row lengths.  Stages below
// k_lo are inactive (dx = 0).  b'_k also goes to ycopy ([K][n]) if given.
// Ends without a barrier after the row sums (the caller syncs).
template <int K>
__device__ void stage_updates(const DevSys& s, const double* __restrict__ b, const double* __restrict__ A,
                              const double* dx, double* part, int cmax, double* bp, double* ycopy, int k, int k_lo,
                              GridBarrier& gb) {
  const int n = s.n, d = s.d, nnz = s.nnz;
  const int gw = gwarp(), nw = nwarps(), lane = lane_id();
  const long long lsV = (long long)d * n;
  const long long lsA = (long long)d * nnz;
  const int kk = k - k_lo;
  if (kk > 0) {
    int maxlen = 0;
    for (int i = lane; i < n; i += 32) maxlen = max(maxlen, s.row_ptr[i + 1] - s.row_ptr[i]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) maxlen = max(maxlen, __shfl_xor_sync(0xffffffffu, maxlen, off));
    const int cpr = (kk * maxlen + UCH - 1) / UCH;  // chunk slots per row
    const long long lsP = (long long)n * cmax;
    for (long long slot = gw; slot < (long long)n * cpr; slot += nw) {
      const int i = (int)(slot / cpr), c = (int)(slot % cpr);
      const int r0 = s.row_ptr[i], len = s.row_ptr[i + 1] - r0;
      const int tot = kk * len;
      if (c * UCH >= tot) continue;  // empty slot (short row), warp-uniform
      md::mdv<K> acc = md::zero<K>();
      for (int t = c * UCH + lane; t < min(tot, (c + 1) * UCH); t += 32) {
        const int j = 1 + t / len;
        const int e = r0 + t % len;
        md::mdv<K> aij = md::load<K>(A + (long long)j * nnz, lsA, e);
        md::mdv<K> xv = md::load_cg<K>(dx + (long long)(k - j) * n, lsV, s.col_idx[e]);
        acc = md::fma_acc<K>(acc, aij, xv);
      }
      acc = md::group_sum<K>(acc, 32);
      if (lane == 0) md::store_cg<K>(part, lsP, (long long)i * cmax + c, acc);
    }
    gb.sync();
    for (int i = gw; i < n; i += nw) {
      const int len = s.row_ptr[i + 1] - s.row_ptr[i];
      const int nc = (kk * len + UCH - 1) / UCH;
      md::mdv<K> acc = md::zero<K>();
      for (int c = lane; c < nc; c += 32) acc = md::add<K>(acc, md::load_cg<K>(part, lsP, (long long)i * cmax + c));
      acc = md::group_sum<K>(acc, 32);
      if (lane == 0) {
        const md::mdv<K> v = md::sub<K>(md::load<K>(b + (long long)k * n, lsV, i), acc);
        md::store_cg<K>(bp + (long long)k * n, lsV, i, v);
        if (ycopy) md::store_cg<K>(ycopy, n, i, v);
      }
    }
  } else {
    for (int i = gw; i < n; i += nw)
      if (lane == 0) {
        const md::mdv<K> v = md::load<K>(b + (long long)k * n, lsV, i);
        md::store_cg<K>(bp + (long long)k * n, lsV, i, v);
        if (ycopy) md::store_cg<K>(ycopy, n, i, v);
      }
  }
}

template <int K>
__global__ void __launch_bounds__(256) stage_kernel(DevSys s, StageArgs a, unsigned* bar) {
  GridBarrier gb(bar, 0u);
  const int n = s.n, d = s.d;
  const int gw = gwarp(), nw = nwarps(), lane = lane_id();
  const long long lsV = (long long)d * n;     // limb stride of [K][d][n]
  const long long lsM = (long long)n * n;
  const int TB = a.TB;
  const int T = (n + TB - 1) / TB;
  const long long lsI = (long long)T * TB * TB;
  for (int k = a.k_lo; k < s.dc; ++k) {
    stage_updates<K>(s, a.b, a.A, a.dx, a.part, a.cmax, a.bp, nullptr, k, a.k_lo, gb);
    gb.sync();
    if (a.M) {
      // ---- dx_k = M b'_k  (qhb and bs in one matvec)
      for (int i = gw; i < n; i += nw) {
        md::mdv<K> acc = md::zero<K>();
        for (int c = lane; c < n; c += 32)
          acc = md::fma_acc<K>(acc, md::load<K>(a.M, lsM, (long long)i * n + c),
                               md::load_cg<K>(a.bp + (long long)k * n, lsV, c));
        acc = md::group_sum<K>(acc, 32);
        if (lane == 0) md::store_cg<K>(a.dx + (long long)k * n, lsV, i, acc);
      }
      gb.sync();
      continue;
    }
    // ---- qhb: y = Q^T b'_k
    for (int i = gw; i < n; i += nw) {
      md::mdv<K> acc = md::zero<K>();
      for (int c = lane; c < n; c += 32) {
        md::mdv<K> q = md::load<K>(a.Qt, lsM, (long long)i * n + c);
        md::mdv<K> v = md::load_cg<K>(a.bp + (long long)k * n, lsV, c);
        acc = md::fma_acc<K>(acc, q, v);
      }
      acc = md::group_sum<K>(acc, 32);
      if (lane == 0) md::store_cg<K>(a.y, n, i, acc);
    }
    gb.sync();
    // ---- bs: tiles last to first
    for (int t = T - 1; t >= 0; --t) {
      const int t0 = t * TB, t1 = min(n, t0 + TB);
      // z_r = y_r - sum_{c >= t1} R[r][c] dx_k[c]   (z kept in y)
      if (t < T - 1) {
        for (int r = t0 + gw; r < t1; r += nw) {
          md::mdv<K> acc = md::zero<K>();
          for (int c = t1 + lane; c < n; c += 32) {
            md::mdv<K> rv = md::load<K>(a.R, lsM, (long long)r * n + c);
            md::mdv<K> xv = md::load_cg<K>(a.dx + (long long)k * n, lsV, c);
            acc = md::fma_acc<K>(acc, rv, xv);
          }
          acc = md::group_sum<K>(acc, 32);
          if (lane == 0) {
            md::mdv<K> yr = md::load_cg<K>(a.y, n, r);
            md::store_cg<K>(a.y, n, r, md::sub<K>(yr, acc));
          }
        }
        gb.sync();
      }
      // dx_k[r] = sum_{c in tile} invR_t[r][c] z_c
      for (int r = t0 + gw; r < t1; r += nw) {
        md::mdv<K> acc = md::zero<K>();
        for (int c = t0 + lane; c < t1; c += 32) {
          md::mdv<K> iv = md::load<K>(a.invR, lsI, (long long)t * TB * TB + (long long)(r - t0) * TB + (c - t0));
          md::mdv<K> zv = md::load_cg<K>(a.y, n, c);
          acc = md::fma_acc<K>(acc, iv, zv);
        }
        acc = md::group_sum<K>(acc, 32);
        if (lane == 0) md::store_cg<K>(a.dx + (long long)k * n, lsV, r, acc);
      }
      gb.sync();
    }
  }
}

// ------------------------------------------------------------------ stage loop, split design
// Right-looking updates off the critical path.  CTAs [0, Q) (the critical
// group, one warp per row) run the dependent chain
//   b'_k = pend_k - A_1 dx_{k-1};  sub-barrier;  dx_k = M b'_k;
//   sub-barrier;  publish dx_k (counter ndx = k + 1)
// while CTAs [Q, G) (the bulk group) apply, as soon as dx_k is published,
//   pend_{k'} -= A_{k'-k} dx_k   for every k' >= k + 2, every row.
// Each (k', row) pair is owned by one bulk warp (lane-held, up to 32 per
// group) that applies k = k_lo, k_lo+1, ... in order, so
// pend_{k'} = b_{k'} - sum_{j >= 2} A_j dx_{k'-j} accumulates in a fixed order
// (deterministic) whatever the timing: lane l of the pair's warp keeps its
// partial sum over the row entries e = l (mod 32) for k = k_lo, k_lo+1, ...
// in a per-pair slot (part), and the warp butterfly runs once, after the
// last k (one md reduction per pair instead of one per (pair, k)); among its pairs with work available
// the warp always takes the most urgent (smallest k').  (Moving the j = 2
// term into the critical chain too was measured slower: the chain's row dots
// are FP64-issue bound, NS_STAGE_TRACE.)
// pdone[k'] counts rows whose pend_{k'} is complete.
struct Stage2Args {
  const double* b;     // [K][d][n]
  const double* A;     // [K][d][nnz]
  const double* M;     // [K][n][n]
  double* bp;          // [K][d][n]   b'_k
  double* dx;          // [K][d][n]
  double* pend;        // [K][d][n]   pending right-hand sides
  int* ndx;            // [1] dx_0..dx_{ndx-1} published (zeroed per launch)
  int* pdone;          // [d] rows of pend_k complete
  unsigned* cbar;      // critical-group barrier counter (zeroed per launch)
  int Q;               // CTAs in the critical group
  int k_lo;            // first active stage (stages below: dx = 0, reading R34); last = s.dc - 1
  long long* tr;       // [d][4] globaltimer stamps of the critical chain (NS_STAGE_TRACE), or nullptr
  double* part;        // [npairs][K][32] per-lane partial sums of the bulk pairs
  int cwpb;            // warps per critical CTA that own a row (warps 0..cwpb-1; <= blockDim / 32)
};

__device__ __forceinline__ void sub_sync(unsigned* cnt, unsigned& target, unsigned nq) {
  __syncthreads();
  target += nq;
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
    while ((int)(ld_relaxed_u32(cnt) - target) < 0) {
    }
    (void)ld_acquire_u32(cnt);
  }
  __syncthreads();
}

template <int K>
__device__ md::mdv<K> row_dot_A(const DevSys& s, const double* A, int j, const double* v, long long lsV, int i) {
  // sum_e A_j[e] v[col e] over the structural entries of row i; warp-wide
  const int lane = threadIdx.x & 31;
  const long long lsA = (long long)s.d * s.nnz;
  const int r0 = s.row_ptr[i], r1 = s.row_ptr[i + 1];
  return warp_dot_levels<K>(r0 + lane, r1, 32, [&](int e, md::mdv<K>& xa, md::mdv<K>& yb) {
    xa = md::load<K>(A + (long long)j * s.nnz, lsA, e);
    yb = md::load_cg<K>(v, lsV, s.col_idx[e]);
  });
}

template <int K>
__global__ void __launch_bounds__(256) stage2_kernel(DevSys s, Stage2Args a, unsigned* bar) {
  const int n = s.n, d = s.d, dc = s.dc, k_lo = a.k_lo;
  const long long lsV = (long long)d * n, lsM = (long long)n * n;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, wpb = blockDim.x >> 5;
  // prologue: pend = b (all CTAs), dx_k = 0 for the retired stages k < k_lo, one full barrier
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < (long long)K * d * n;
       t += (long long)gridDim.x * blockDim.x) {
    __stcg(a.pend + t, a.b[t]);
    if ((int)((t / n) % d) < k_lo) __stcg(a.dx + t, 0.0);
  }
  {
    GridBarrier gb(bar, 0u);
    gb.sync();
  }
  if ((int)blockIdx.x < a.Q) {
    // ---------------- critical group
    // warps 0..cwpb-1 own rows (cwpb = 4: one row-owning warp per SMSP, so a row dot
    // does not share its SMSP's FP64 pipe with another one); the rest only join the barriers
    const int cw = (wib < a.cwpb) ? blockIdx.x * a.cwpb + wib : n, ncw = a.Q * a.cwpb;
    unsigned target = 0;
    const bool trc = a.tr && blockIdx.x == 0 && threadIdx.x == 0;
    // Each critical warp owns at most one row (ncw >= n).  The stage-invariant
    // operands of its two dots -- row i of A_1 with its column indices and row
    // i of M -- stay in registers for the whole loop (lane l holds entries
    // l + 32 q), so a stage only loads dx_{k-1} and b'_k.  Same term order as
    // the streamed path (dot_ilp<K, 1>), so the results are identical.
    // (not at 8d: the cached operands cost spills there; C3 measured 22 vs 17 us per dot)
    constexpr int RQ = 2;  // n <= 64 (C2)
    const int row = cw;
    int r0 = 0, len = 0;
    if (row < n) {
      r0 = s.row_ptr[row];
      len = s.row_ptr[row + 1] - r0;
    }
    // grid-uniform choice (every critical warp takes the same path, so every
    // thread reaches the same sub_sync barrier instructions); warps without a
    // row (row >= n) run the cached path with no loads and no stores
    int maxlen = 0;
    for (int r = lane; r < n; r += 32) maxlen = max(maxlen, s.row_ptr[r + 1] - s.row_ptr[r]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) maxlen = max(maxlen, __shfl_xor_sync(0xffffffffu, maxlen, off));
    const bool cache = K < 8 && n <= 32 * RQ && maxlen <= 32 * RQ;
    const bool has_row = row < n;
    md::mdv<K> a1c[RQ], mc[RQ];
    int colc[RQ];
    if (cache) {
      const long long lsA = (long long)d * s.nnz;
#pragma unroll
      for (int q = 0; q < RQ; ++q) {
        const int t = lane + 32 * q;
        a1c[q] = (t < len) ? md::load<K>(a.A + s.nnz, lsA, r0 + t) : md::zero<K>();
        colc[q] = (t < len) ? s.col_idx[r0 + t] : 0;
        mc[q] = (has_row && t < n) ? md::load<K>(a.M, lsM, (long long)row * n + t) : md::zero<K>();
      }
    }
    for (int k = k_lo; k < dc; ++k) {
      if (trc) a.tr[4 * k] = gtimer();
      if (k >= k_lo + 2) {
        if (threadIdx.x == 0) flag_wait(a.pdone + k, n);
        __syncthreads();
      }
      if (trc) a.tr[4 * k + 1] = gtimer();
      if (cache) {
        md::mdv<K> v = has_row ? md::load_cg<K>(a.pend + (long long)k * n, lsV, row) : md::zero<K>();
        if (k >= k_lo + 1) {
          const double* xp = a.dx + (long long)(k - 1) * n;
          md::mdv<K> xv[RQ];
#pragma unroll
          for (int q = 0; q < RQ; ++q) xv[q] = (lane + 32 * q < len) ? md::load_cg<K>(xp, lsV, colc[q]) : md::zero<K>();
          double sl[K];
#pragma unroll
          for (int l = 0; l < K; ++l) sl[l] = 0.0;
#pragma unroll
          for (int q = 0; q < RQ; ++q)
            if (lane + 32 * q < len) {
              double pl[K];
              md::prod_levels<K>(a1c[q], xv[q], pl);
#pragma unroll
              for (int l = 0; l < K; ++l) md::level_insert<K>(sl, l, pl[l]);
            }
          v = md::sub<K>(v, md::group_sum_levels<K>(sl, 32));
        }
        if (lane == 0 && has_row) md::store_cg<K>(a.bp + (long long)k * n, lsV, row, v);
        sub_sync(a.cbar, target, a.Q);
        if (trc) a.tr[4 * k + 2] = gtimer();
        const double* bk = a.bp + (long long)k * n;
        md::mdv<K> bv[RQ];
#pragma unroll
        for (int q = 0; q < RQ; ++q) bv[q] = (lane + 32 * q < n) ? md::load_cg<K>(bk, lsV, lane + 32 * q) : md::zero<K>();
        double sl[K];
#pragma unroll
        for (int l = 0; l < K; ++l) sl[l] = 0.0;
#pragma unroll
        for (int q = 0; q < RQ; ++q)
          if (lane + 32 * q < n) {
            double pl[K];
            md::prod_levels<K>(mc[q], bv[q], pl);
#pragma unroll
            for (int l = 0; l < K; ++l) md::level_insert<K>(sl, l, pl[l]);
          }
        const md::mdv<K> acc = md::group_sum_levels<K>(sl, 32);
        if (lane == 0 && has_row) md::store_cg<K>(a.dx + (long long)k * n, lsV, row, acc);
        sub_sync(a.cbar, target, a.Q);
        if (trc) a.tr[4 * k + 3] = gtimer();
        if (blockIdx.x == 0 && threadIdx.x == 0) flag_set(a.ndx, k + 1);
        continue;
      }
      for (int i = cw; i < n; i += ncw) {
        md::mdv<K> v = md::load_cg<K>(a.pend + (long long)k * n, lsV, i);
        if (k >= k_lo + 1)
          v = md::sub<K>(v, row_dot_A<K>(s, a.A, 1, a.dx + (long long)(k - 1) * n, lsV, i));
        if (lane == 0) md::store_cg<K>(a.bp + (long long)k * n, lsV, i, v);
      }
      sub_sync(a.cbar, target, a.Q);
      if (trc) a.tr[4 * k + 2] = gtimer();
      for (int r = cw; r < n; r += ncw) {
        const md::mdv<K> acc = warp_dot_levels<K>(lane, n, 32, [&](int c, md::mdv<K>& xa, md::mdv<K>& yb) {
          xa = md::load<K>(a.M, lsM, (long long)r * n + c);
          yb = md::load_cg<K>(a.bp + (long long)k * n, lsV, c);
        });
        if (lane == 0) md::store_cg<K>(a.dx + (long long)k * n, lsV, r, acc);
      }
      sub_sync(a.cbar, target, a.Q);
      if (trc) a.tr[4 * k + 3] = gtimer();
      if (blockIdx.x == 0 && threadIdx.x == 0) flag_set(a.ndx, k + 1);
    }
  } else {
    // ---------------- bulk group: (k', i) pairs, k' = k_lo+2..dc-1; a warp holds up to 32
    // pairs (one per lane, ascending k') and always serves the most urgent one with work.
    // Work unit = one 32-entry chunk of row i for one k (one fused multiply-add per lane),
    // so a newly urgent pair waits for at most one chunk, not a whole row dot.  Units of a
    // pair run in the order (k ascending, chunk ascending); the lane partials stay in
    // registers while the warp keeps serving the same pair and go to the pair's slot
    // (part) when it switches.
    const int bw = (blockIdx.x - a.Q) * wpb + wib, nbw = ((int)gridDim.x - a.Q) * wpb;
    const int npairs = (dc - 2 - k_lo) * n;
    const long long lsA = (long long)d * s.nnz;
    int avail = 0;  // dx published so far (this warp's view)
    for (int g0 = bw; g0 < npairs; g0 += 32 * nbw) {
      const int p = g0 + lane * nbw;
      const bool has = p < npairs;
      const int kp = has ? k_lo + 2 + p / n : 0, i = has ? p % n : 0;
      const int len = has ? s.row_ptr[i + 1] - s.row_ptr[i] : 0;
      const int nch = max(1, (len + 31) / 32);
      const int units = has ? (kp - 1 - k_lo) * nch : 0;  // k = k_lo..kp-2, nch chunks each
      int pu = 0;                                          // units done
      bool live = units > 0;
      int cur = -1;  // pair whose lane partials are in acc (warp-uniform)
      md::mdv<K> acc = md::zero<K>();
      for (;;) {
        if (!__any_sync(0xffffffffu, live)) break;
        // refresh the published count every round (a stale count would hide a
        // newly urgent pair behind the backlog of less urgent work)
        if (lane == 0 && ld_relaxed_s32(a.ndx) > avail) avail = ld_acquire(a.ndx);
        avail = __shfl_sync(0xffffffffu, avail, 0);
        __syncwarp();  // orders the other lanes' dx loads after lane 0's acquire (a shuffle does not)
        const unsigned m = __ballot_sync(0xffffffffu, live && k_lo + pu / nch < avail);
        if (m == 0) {  // nothing available: wait for the next dx
          if (lane == 0) {
            while (ld_relaxed_s32(a.ndx) <= avail) {
            }
            avail = ld_acquire(a.ndx);
          }
          avail = __shfl_sync(0xffffffffu, avail, 0);
          __syncwarp();
          continue;
        }
        const int src = __ffs(m) - 1;
        const int skp = __shfl_sync(0xffffffffu, kp, src), si = __shfl_sync(0xffffffffu, i, src);
        const int spu = __shfl_sync(0xffffffffu, pu, src), sp = __shfl_sync(0xffffffffu, p, src);
        const int snch = __shfl_sync(0xffffffffu, nch, src), sunits = __shfl_sync(0xffffffffu, units, src);
        const int sk = k_lo + spu / snch, sch = spu % snch;
        if (sp != cur) {  // switch pairs: park the current partials, fetch the new ones
          if (cur >= 0) {
            double* slot = a.part + (long long)cur * K * 32 + lane;
#pragma unroll
            for (int l = 0; l < K; ++l) slot[32 * l] = acc.x[l];
          }
          if (spu == 0) {
            acc = md::zero<K>();
          } else {
            const double* slot = a.part + (long long)sp * K * 32 + lane;
#pragma unroll
            for (int l = 0; l < K; ++l) acc.x[l] = slot[32 * l];
          }
          cur = sp;
        }
        {
          const int e = s.row_ptr[si] + sch * 32 + lane;
          if (e < s.row_ptr[si + 1]) {  // acc holds unnormalised level sums (no renormalisation per term)
            double pl[K];
            md::prod_levels<K>(md::load<K>(a.A + (long long)(skp - sk) * s.nnz, lsA, e),
                               md::load_cg<K>(a.dx + (long long)sk * n, lsV, s.col_idx[e]), pl);
#pragma unroll
            for (int l = 0; l < K; ++l) md::level_insert<K>(acc.x, l, pl[l]);
          }
        }
        if (spu == sunits - 1) {  // last unit of pend_{k'} row i: reduce the lanes once
          const md::mdv<K> tot = md::group_sum_levels<K>(acc.x, 32);
          if (lane == 0) {
            const long long e = (long long)skp * n;
            md::store_cg<K>(a.pend + e, lsV, si, md::sub<K>(md::load_cg<K>(a.pend + e, lsV, si), tot));
            if (a.tr) {  // trace: when the last row of pend_{k'} completes, and the unit count
              __threadfence();
              if (atomicAdd(a.pdone + skp, 1) == n - 1) a.tr[4 * d + skp] = gtimer();
            } else {
              asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(a.pdone + skp) : "memory");
            }
          }
          cur = -1;
        }
        if (lane == src) {
          ++pu;
          live = pu < units;
        }
      }
    }
  }
}

// ------------------------------------------------------------------ residual and norms
// r_k,i = b'_k,i - sum_c A0[i][c] dx_k[c]: warps over all (k, i) rows of the grid.
template <int K>
__global__ void __launch_bounds__(256) residual_kernel(int n, int d, int dc, int k_lo, const int* __restrict__ rows,
                                                       int nr, const double* __restrict__ b,
                                                       const double* __restrict__ bp,
                                                       const double* __restrict__ A0,
                                                       const double* __restrict__ dx, double* rbuf,
                                                       double* knorm) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  const long long lsV = (long long)d * n, lsM = (long long)n * n;
  // rows: the sampled equations (NEXT-4), nr of them; nullptr = all n
  for (long long row = gw; row < (long long)dc * nr; row += nw) {
    const int k = (int)(row / nr), i = rows ? rows[row % nr] : (int)(row % nr);
    md::mdv<K> acc = md::zero<K>();
    if (k >= k_lo)  // warp-uniform (row is per warp)
      acc = warp_dot_levels<K>(lane, n, 32, [&](int c, md::mdv<K>& xa, md::mdv<K>& yb) {
        xa = md::load<K>(A0, lsM, (long long)i * n + c);
        yb = md::load<K>(dx + (long long)k * n, lsV, c);
      });
    if (lane == 0) {
      md::mdv<K> r = (k >= k_lo) ? md::sub<K>(md::load<K>(bp + (long long)k * n, lsV, i), acc)
                                 : md::load<K>(b + (long long)k * n, lsV, i);
      md::store<K>(rbuf + (long long)k * n, lsV, i, r);
    }
  }
}

// knorm[w][k] = sum_i |v_k,i| for v = b, r, dx, x (one CTA per active k, one warp
// per norm; x is the series before the update, [K][n][d])
template <int K>
__global__ void __launch_bounds__(128) knorm_kernel(int n, int d, int k_lo, const int* __restrict__ rows, int nr,
                                                    const double* __restrict__ b,
                                                    const double* __restrict__ rbuf, const double* __restrict__ dx,
                                                    const double* __restrict__ x, double* knorm) {
  const int k = blockIdx.x, w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long lsV = (long long)d * n;
  const double* src = (w == 0) ? b : ((w == 1) ? rbuf : dx);
  md::mdv<K> acc = md::zero<K>();
  // the residual norm runs over the sampled equations; rbuf = nullptr
  // (NS_NO_RESIDUAL): no residual, its norm is 0
  const int cnt = (w == 1) ? (rbuf ? nr : 0) : n;
  for (int t = lane; t < cnt; t += 32) {
    const int i = (w == 1 && rows) ? rows[t] : t;
    md::mdv<K> v = (w == 3) ? md::load<K>(x, lsV, (long long)i * d + k) : md::load<K>(src + (long long)k * n, lsV, i);
    if (w == 2 && k < k_lo) v = md::zero<K>();
    acc = md::add<K>(acc, md::absv<K>(v));
  }
  acc = md::group_sum<K>(acc, 32);
  if (lane == 0) md::store<K>(knorm + (long long)w * K * d, d, k, acc);
}

// Fabry ratio (NEXT-4; Theorem 1 P:194-208 and its numerical interpretation
// P:210-219): z_j = c_{D-1} / c_D of the series x_j, an estimate of the
// nearest singularity (|z_j| = radius of convergence); c_D = 0 gives +inf.
template <int K>
__global__ void fabry_kernel(int n, int d, const double* __restrict__ x, double* z) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const long long lsX = (long long)n * d;
  const md::mdv<K> a = md::load<K>(x, lsX, (long long)j * d + d - 2);
  const md::mdv<K> c = md::load<K>(x, lsX, (long long)j * d + d - 1);
  md::mdv<K> r;
  if (md::is_zero<K>(c)) {
    r = md::zero<K>();
    r.x[0] = __longlong_as_double(0x7ff0000000000000LL);  // +inf
  } else {
    r = md::div<K>(a, c);
  }
  md::store<K>(z, n, j, r);
}

// x += dx (one thread per coefficient); warp 0 of block 0 reduces the norms.
template <int K>
__global__ void finalize_kernel(int n, int d, int dc, double* x, const double* __restrict__ dx,
                                const double* __restrict__ knorm, double* res_out, unsigned* status) {
  const long long lsX = (long long)n * d, lsV = (long long)d * n;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < (long long)n * d;
       t += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(t / d), k = (int)(t % d);
    if (k >= dc) continue;  // outside the window: x_k unchanged
    md::mdv<K> xv = md::load<K>(x, lsX, t);
    md::mdv<K> dv = md::load<K>(dx + (long long)k * n, lsV, j);
    md::store<K>(x, lsX, t, md::add<K>(xv, dv));
  }
  if (blockIdx.x == 0 && threadIdx.x < 96) {
    // warp w: max over k of knorm[w][k]; lanes stride k, then a shuffle max
    // (a max is exact, so the order does not matter)
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    md::mdv<K> best = md::zero<K>();
    bool nonfinite = false;
    for (int k = lane; k < dc; k += 32) {
      const md::mdv<K> v = md::load<K>(knorm + (long long)w * K * d, d, k);
      nonfinite |= !isfinite(v.x[0]);
      if (md::greater<K>(v, best)) best = v;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const md::mdv<K> o = md::shfl_xor<K>(best, off);
      if (md::greater<K>(o, best)) best = o;
    }
    nonfinite = __any_sync(0xffffffffu, nonfinite);
    if (lane == 0) {
      md::store<K>(res_out, 3, w, best);
      if (nonfinite || !isfinite(best.x[0])) atomicOr(status, ST_NONFINITE);
    }
  }
}

}  // namespace ns
