// cqr.cuh -- Householder QR of [A_0 | I] inside ONE thread-block cluster
// (same arithmetic as householder_qr_kernel
// in solve.cuh, different machine mapping).
//
// Why a cluster: the QR is a chain of n dependent steps (reflector j needs
// column j after reflectors 0..j-1), each a few md operations long.  With the
// grid-wide kernel every step pays two L2 flag round trips plus L2 loads of the
// reflector; here the 2n columns live in the shared memory of the P CTAs of
// one cluster and each reflector is pushed into every CTA's shared memory
// (DSMEM stores) and signalled with mbarriers, so a step costs one DSMEM
// round trip instead of ~4 L2 round trips, and nothing on the critical path
// touches L2 (immune to the concurrent eval/diff kernel's traffic).
//
// Mapping: column c (0..2n-1) lives in CTA c % P, local slot c / P; warp w of a
// CTA owns local slots w, w + W (at most CPW = 2).  Reflector j (rows j..n-1)
// goes into ring slot j % RS of every CTA in two parts:
//   A part (fullA[s], 32 arrivals): rows > j of v_j = the final rows > j of
//          column j; published by the owner of column j as soon as its column
//          is updated, so every warp forms its partial dot sum_{r>j} v_r a_r
//          while the owner still computes the norm, sqrt and alpha v0;
//   B part (fullB[s], 1 arrival): v0 = a_jj - alpha; consumers add v0 a_j to
//          their partial dots while the owner forms beta = -1 / (alpha v0);
//   C part (fullC[s], 1 arrival): beta (one reciprocal per reflector, not one
//          per consumer warp: the consumer warps share the SMs' FP64 pipes).
// A slot is rewritten only after every warp of the cluster has finished the
// step that used it (empty[s]: P W arrivals, one per warp after __syncwarp,
// waited on by the writer).
// The owner of column j+1 applies H_j to it first and builds reflector j+1 at
// once (look-ahead of one column): the critical path per step is one column
// update + one reflector + one DSMEM hop.
//
// Output: R (row-major, upper; R_jj = alpha_j), Q^T (row-major), rdiag, and the
// singular flag, exactly what qr_unpack_kernel produced from W.
#pragma once
#include "common.cuh"
#include "evaldiff.cuh"

namespace ns {
namespace cq {

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned mapa(unsigned addr, unsigned rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_remote(unsigned addr, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
}
__device__ __forceinline__ void arrive_remote(unsigned bar_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_addr) : "memory");
}
__device__ __forceinline__ void bar_init(unsigned bar_addr, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar_addr), "r"(count) : "memory");
}
__device__ __forceinline__ void bar_wait(unsigned bar_addr, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar_addr),
      "r"(parity)
      : "memory");
}
// Transfers complete on the DESTINATION's mbarrier (complete_tx); each
// destination CTA arms its own barrier for the phase with a local
// arrive.expect_tx (arm), so a producer never waits on a remote arrival.
__device__ __forceinline__ void arm(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
// bulk copy (async proxy) of `bytes` from this CTA's shared memory into CTA
// `rank`'s shared memory at the same offset as dst_local
__device__ __forceinline__ void bulk_push(unsigned dst_local, unsigned src, unsigned bytes, unsigned bar_local,
                                          unsigned rank) {
  const unsigned dst = mapa(dst_local, rank), bar = mapa(bar_local, rank);
  asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "r"(src), "r"(bytes), "r"(bar)
               : "memory");
}
// two doubles into CTA `rank`'s shared memory (st.async: no proxy fence needed)
__device__ __forceinline__ void st_async2(unsigned dst_local, double a, double b, unsigned bar_local, unsigned rank) {
  const unsigned dst = mapa(dst_local, rank), bar = mapa(bar_local, rank);
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(dst), "d"(a),
               "d"(b), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

// sum over the rows r > j held by this lane (rows lane + 32 q) of a_r b_r, as
// unnormalised levels, reduced over the warp (md::group_sum_levels)
template <int K, int E>
MD_INL md::mdv<K> dot_tail(const double* a, const double* b, int n, int j) {
  const int lane = threadIdx.x & 31;
  double s[K];
#pragma unroll
  for (int l = 0; l < K; ++l) s[l] = 0.0;
#pragma unroll
  for (int q = 0; q < E; ++q) {
    const int r = lane + 32 * q;
    if (r > j && r < n) {
      double p[K];
      md::prod_levels<K>(md::load<K>(a, n, r), md::load<K>(b, n, r), p);
#pragma unroll
      for (int l = 0; l < K; ++l) md::level_insert<K>(s, l, p[l]);
    }
  }
  return md::group_sum_levels<K>(s, 32);
}

}  // namespace cq

// Shared-memory layout (doubles): cols [CPC][K][n], vt [RS][K][n] (reflector
// rows), sc [RS][2][K] (v0, beta), stg [RS][2][K] (unused), then 4 RS + 1
// mbarriers.  Rows go with one bulk copy per destination CTA, v0 and beta with
// st.async; both complete on the destination's barrier.
// With withM, R is broadcast to every CTA (Rs [n][K][n], column-major like
// cols, and rinv [K][n]) and the warps owning the columns of Q^T back-substitute
// them: M = R^{-1} Q^T leaves the cluster directly (no invert / form_m kernels).
struct CqrShape {
  int P, W, CPC, RS, withM;
};
__host__ __device__ inline size_t cqr_smem_bytes(int n, int K, const CqrShape& sh) {
  size_t dbl = (size_t)sh.CPC * K * n + (size_t)sh.RS * K * n + 2 * (size_t)sh.RS * 2 * K;
  if (sh.withM) dbl += (size_t)n * K * n + (size_t)K * n;
  return dbl * sizeof(double) + (4 * (size_t)sh.RS + 1) * sizeof(unsigned long long);
}

template <int K, int E>
__global__ void __launch_bounds__(K == 8 ? 256 : 512) cluster_qr_kernel(DevSys sy, const double* __restrict__ x, int n,
                                                         const double* __restrict__ A0, double* Wg, double* R,
                                                         double* Qt, double* rdiag, unsigned* status,
                                                         CqrShape sh, long long* tr, double* Mout) {
  // tr (debug, nullptr normally): [n][8] globaltimer stamps of the look-ahead warp
  constexpr int CPW = 2;
  extern __shared__ __align__(16) double cq_sm[];
  const int P = sh.P, W = sh.W, CPC = sh.CPC, RS = sh.RS;
  const int ncol = 2 * n;
  const unsigned rank = cq::cluster_rank();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* cols = cq_sm;
  double* vt = cols + (size_t)CPC * K * n;
  double* sc = vt + (size_t)RS * K * n;
  double* stg = sc + (size_t)RS * 2 * K;
  double* Rs = stg + (size_t)RS * 2 * K;                       // withM: [n][K][n]
  double* rinv = Rs + (sh.withM ? (size_t)n * K * n : 0);      // withM: [K][n]
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(rinv + (sh.withM ? (size_t)K * n : 0));
  const unsigned rfull = cq::smem_u32(bars + 4 * RS);
  const unsigned fullA0 = cq::smem_u32(bars), fullB0 = cq::smem_u32(bars + RS), empty0 = cq::smem_u32(bars + 2 * RS),
                 fullC0 = cq::smem_u32(bars + 3 * RS);
  const unsigned vt0 = cq::smem_u32(vt), sc0 = cq::smem_u32(sc);
  auto col_ptr = [&](int lc) { return cols + (size_t)lc * K * n; };
  // phase stamps (trace only) in the unused look-ahead row n-1: start, columns
  // loaded, steps done, R/Q^T written, M written
  long long* ph_tr = (tr && rank == 0 && threadIdx.x == 0) ? tr + 8LL * (n - 1) : nullptr;
  if (ph_tr) ph_tr[0] = gtimer();

  // ---- A_0 (formed from x by warp per equation into W, or read from A0) and I
  if (x) {
    const int gw = (int)rank * W + warp, nw = P * W;
    for (int i = gw; i < n; i += nw) a0_row<K>(sy, x, i, Wg, (long long)n * n, 1, n);  // W[l][c][r]
  }
  if (threadIdx.x == 0) {
    for (int q = 0; q < RS; ++q) {
      cq::bar_init(fullA0 + 8 * q, 1);  // the local arm; the bytes come with the copies
      cq::bar_init(fullB0 + 8 * q, 1);
      cq::bar_init(fullC0 + 8 * q, 1);
      cq::bar_init(empty0 + 8 * q, (unsigned)(P * W));
    }
    cq::bar_init(rfull, 1u);
  }
  const unsigned bytesA = (unsigned)(K * n * sizeof(double)), bytesS = (unsigned)(K * sizeof(double));
  // thread 0 arms every slot's A/B/C barriers one phase (step) ahead
  auto arm_step = [&](int j) {
    const int s = j % RS;
    cq::arm(fullA0 + 8 * s, bytesA);
    cq::arm(fullB0 + 8 * s, bytesS);
    cq::arm(fullC0 + 8 * s, bytesS);
  };
  if (threadIdx.x == 0) {
    for (int j = 0; j < RS && j < n; ++j) arm_step(j);
    if (sh.withM) cq::arm(rfull, (unsigned)n * bytesA);  // one bulk copy per R column
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  cq::cluster_sync_all();  // A_0 rows in W visible to the cluster, barriers initialised
  for (int e = threadIdx.x; e < CPC * n; e += blockDim.x) {
    const int lc = e / n, r = e % n;
    const int c = (int)rank + P * lc;
    double* cp = col_ptr(lc);
#pragma unroll
    for (int l = 0; l < K; ++l) {
      double v = 0.0;
      if (c < n) v = x ? __ldcg(Wg + ((size_t)l * n + c) * n + r) : A0[((size_t)l * n + r) * n + c];
      else if (c < ncol) v = (l == 0 && r == c - n) ? 1.0 : 0.0;
      cp[(size_t)l * n + r] = v;
    }
  }
  __syncthreads();
  if (ph_tr) ph_tr[1] = gtimer();

  // ---- publishing helpers (called by the whole owner warp)
  // A part of reflector jj: the whole column (rows > jj are v; consumers read
  // only those) into vt[s] of every CTA, one bulk copy per CTA (lane p -> CTA p)
  auto publish_A = [&](int jj, const double* cp) {
    const int s = jj % RS;
    cq::fence_proxy_async();  // this lane's column writes -> async proxy
    __syncwarp();
    const unsigned bytes = (unsigned)(K * n * sizeof(double));
    for (int p = lane; p < P; p += 32)
      cq::bulk_push(vt0 + (unsigned)((size_t)s * K * n * sizeof(double)), cq::smem_u32(cp), bytes, fullA0 + 8 * s, p);
  };
  // B part (v0) or C part (beta) of reflector jj to every CTA (lane p -> CTA p)
  auto publish_sc = [&](int jj, int part, const md::mdv<K>& v, unsigned bar0) {
    const int s = jj % RS;
    const unsigned dst = sc0 + (unsigned)(((size_t)s * 2 + part) * K * sizeof(double));
    for (int p = lane; p < P; p += 32) {
#pragma unroll
      for (int l = 0; l < K; l += 2) cq::st_async2(dst + l * sizeof(double), v.x[l], v.x[l + 1], bar0 + 8 * s, p);
    }
  };
  // reflector jj from the (already updated) column: sig = sum_{r >= jj} a_r^2
  auto reflect = [&](int jj, double* cp, const md::mdv<K>& sig) {
    const md::mdv<K> x0 = md::load<K>(cp, n, jj);  // warp-uniform smem read
    const md::mdv<K> nrm = md::sqrt<K>(sig);
    const md::mdv<K> alpha = md::is_negative<K>(x0) ? nrm : md::neg<K>(nrm);  // reading R13
    const md::mdv<K> v0 = md::sub<K>(x0, alpha);
    publish_sc(jj, 0, v0, fullB0);
    // v^T v = -2 alpha v0, beta = 2 / v^T v = -1 / (alpha v0); zero column: beta = 0 (H = I)
    md::mdv<K> bt = md::zero<K>();
    if (!md::is_zero<K>(sig)) bt = md::neg<K>(md::recip<K>(md::mul<K>(alpha, v0)));
    else if (lane == 0 && status) atomicOr(status, ST_SINGULAR);
    publish_sc(jj, 1, bt, fullC0);
    __syncwarp();
    if (lane == 0) md::store<K>(cp, n, jj, alpha);  // R_jj (rows > jj keep v, unused)
    if (lane == 0) md::store<K>(rdiag, n, jj, alpha);
  };

  // ---- reflector 0 (owner of column 0: CTA 0, warp 0)
  if (rank == 0 && warp == 0) {
    double* cp = col_ptr(0);
    publish_A(0, cp);
    md::mdv<K> sig;
    {
      double s[K];
#pragma unroll
      for (int l = 0; l < K; ++l) s[l] = 0.0;
#pragma unroll
      for (int q = 0; q < E; ++q) {
        const int r = lane + 32 * q;
        if (r < n) {
          const md::mdv<K> a = md::load<K>(cp, n, r);
          double pl[K];
          md::prod_levels<K>(a, a, pl);
#pragma unroll
          for (int l = 0; l < K; ++l) md::level_insert<K>(s, l, pl[l]);
        }
      }
      sig = md::group_sum_levels<K>(s, 32);
    }
    reflect(0, cp, sig);
  }

  // ---- steps
  for (int j = 0; j < n; ++j) {
    const int s = j % RS;
    const unsigned ph = (unsigned)((j / RS) & 1);
    // this warp's active columns (c > j) form a suffix of its slots q = 0..CPW-1
    bool act[CPW];
#pragma unroll
    for (int q = 0; q < CPW; ++q) {
      const int lc = warp + q * W;
      const int c = (int)rank + P * lc;
      act[q] = lc < CPC && c < ncol && c > j;
    }
    const double* vs = vt + (size_t)s * K * n;
    const bool trw = tr && lane == 0 && (act[0] || act[CPW - 1]) &&
                     ((int)rank + P * (act[0] ? warp : warp + W)) == j + 1 && j + 1 < n;
    if (trw) tr[8 * j + 0] = gtimer();
    cq::bar_wait(fullA0 + 8 * s, ph);
    if (trw) tr[8 * j + 1] = gtimer();
    md::mdv<K> part[CPW];
#pragma unroll
    for (int q = 0; q < CPW; ++q)
      if (act[q]) part[q] = cq::dot_tail<K, E>(vs, col_ptr(warp + q * W), n, j);
    if (trw) tr[8 * j + 2] = gtimer();
    cq::bar_wait(fullB0 + 8 * s, ph);
    if (trw) tr[8 * j + 3] = gtimer();
    if (act[0] || act[CPW - 1]) {
      const md::mdv<K> v0 = md::load<K>(sc + (size_t)s * 2 * K, 1, 0);
      md::mdv<K> dots[CPW];
#pragma unroll
      for (int q = 0; q < CPW; ++q)
        if (act[q]) dots[q] = md::fma_acc<K>(part[q], v0, md::load<K>(col_ptr(warp + q * W), n, j));
      cq::bar_wait(fullC0 + 8 * s, ph);
      if (trw) tr[8 * j + 4] = gtimer();
      const md::mdv<K> bt = md::load<K>(sc + (size_t)s * 2 * K + K, 1, 0);
#pragma unroll
      for (int q = 0; q < CPW; ++q) {
        if (act[q]) {
          double* cp = col_ptr(warp + q * W);
          const int c = (int)rank + P * (warp + q * W);
          const md::mdv<K> nw = md::neg<K>(md::mul<K>(bt, dots[q]));
          const bool look = (c == j + 1 && c < n);
          double sg[K];
#pragma unroll
          for (int l = 0; l < K; ++l) sg[l] = 0.0;
#pragma unroll
          for (int qq = 0; qq < E; ++qq) {
            const int r = lane + 32 * qq;
            if (r >= j && r < n) {
              const md::mdv<K> v = (r == j) ? v0 : md::load<K>(vs, n, r);
              const md::mdv<K> w = md::fma_acc<K>(md::load<K>(cp, n, r), nw, v);
              md::store<K>(cp, n, r, w);
              if (look && r > j) {  // look-ahead norm in the same pass
                double pl[K];
                md::prod_levels<K>(w, w, pl);
#pragma unroll
                for (int l = 0; l < K; ++l) md::level_insert<K>(sg, l, pl[l]);
              }
            }
          }
          if (look) {
            const int jj = j + 1;
            if (trw) tr[8 * j + 5] = gtimer();
            if (jj >= RS) cq::bar_wait(empty0 + 8 * (jj % RS), (unsigned)(((jj / RS) - 1) & 1));
            __syncwarp();
            publish_A(jj, cp);
            if (trw) tr[8 * j + 6] = gtimer();
            const md::mdv<K> sig = md::group_sum_levels<K>(sg, 32);
            reflect(jj, cp, sig);
            if (trw) tr[8 * j + 7] = gtimer();
          }
        }
      }
    }
    if (!(act[0] || act[CPW - 1])) cq::bar_wait(fullC0 + 8 * s, ph);  // one arrival per phase
    if (threadIdx.x == 0 && j + RS < n) arm_step(j + RS);  // this CTA's slot s is consumed by warp 0
    __syncwarp();
    // done with slot s: one arrival per warp on every CTA's empty[s]
    for (int p = lane; p < P; p += 32) cq::arrive_remote(cq::mapa(empty0 + 8 * s, p));
  }
  __syncthreads();
  if (ph_tr) ph_tr[2] = gtimer();

  // ---- output: R (row-major upper, diagonal alpha), Q^T (row-major)
  for (int e = threadIdx.x; e < CPC * n; e += blockDim.x) {
    const int lc = e / n, r = e % n;
    const int c = (int)rank + P * lc;
    const double* cp = col_ptr(lc);
#pragma unroll
    for (int l = 0; l < K; ++l) {
      const double v = cp[(size_t)l * n + r];
      if (c < n) R[((size_t)l * n + r) * n + c] = (r <= c) ? v : 0.0;
      else if (c < ncol) Qt[((size_t)l * n + r) * n + (c - n)] = v;
    }
  }
  if (ph_tr) ph_tr[3] = gtimer();
  if (sh.withM && Mout) {
    // R columns (rows <= c final, R_cc = alpha_c) into every CTA's Rs
    cq::fence_proxy_async();
    __syncthreads();
    for (int lc = warp; lc < CPC; lc += W) {
      const int c = (int)rank + P * lc;
      if (c < n)
        for (int p = lane; p < P; p += 32)
          cq::bulk_push(cq::smem_u32(Rs + (size_t)c * K * n), cq::smem_u32(col_ptr(lc)), bytesA, rfull, p);
    }
    cq::bar_wait(rfull, 0);
    // rinv_k = 1 / R_kk, then R'[r][k] = R[r][k] rinv_k (r < k): the chain below
    // is one fused multiply-add per row instead of a multiply and an add
    for (int k = warp; k < n; k += W) {
      const md::mdv<K> rv = md::recip<K>(md::load<K>(Rs + (size_t)k * K * n, n, k));
      if (lane == 0) md::store<K>(rinv, n, k, rv);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
      const int k = e / n, r = e % n;
      if (r < k) {
        double* base = Rs + (size_t)k * K * n;
        md::store<K>(base, n, r, md::mul<K>(md::load<K>(base, n, r), md::load<K>(rinv, n, k)));
      }
    }
    __syncthreads();
    // column i of M = R^{-1} (column n+i of the work matrix, = Q^T e_i): with
    // y = D^{-1} ... the scaled recurrence q_r -= q_k R'[r][k] (k = n-1..0),
    // then m_r = q_r rinv_r
#pragma unroll
    for (int q = 0; q < CPW; ++q) {
      const int lc = warp + q * W;
      const int c = (int)rank + P * lc;
      if (lc < CPC && c >= n && c < ncol) {
        const double* cp = col_ptr(lc);
        md::mdv<K> qv[E];
#pragma unroll
        for (int qq = 0; qq < E; ++qq) {
          const int r = lane + 32 * qq;
          qv[qq] = (r < n) ? md::load<K>(cp, n, r) : md::zero<K>();
        }
        for (int k = n - 1; k > 0; --k) {
          md::mdv<K> qk = qv[0];
#pragma unroll
          for (int qq = 1; qq < E; ++qq)
            if ((k >> 5) == qq) qk = qv[qq];
          qk = md::neg<K>(md::shfl<K>(qk, k & 31));
          const double* Rk = Rs + (size_t)k * K * n;
#pragma unroll
          for (int qq = 0; qq < E; ++qq) {
            const int r = lane + 32 * qq;
            if (r < k) qv[qq] = md::fma_acc<K>(qv[qq], qk, md::load<K>(Rk, n, r));
          }
        }
        const int i = c - n;
#pragma unroll
        for (int qq = 0; qq < E; ++qq) {
          const int r = lane + 32 * qq;
          if (r < n) md::store<K>(Mout + (size_t)r * n + i, (long long)n * n, 0,
                                  md::mul<K>(qv[qq], md::load<K>(rinv, n, r)));
        }
      }
    }
  }
  if (ph_tr) ph_tr[4] = gtimer();
  cq::cluster_sync_all();  // no CTA leaves while DSMEM traffic to it may be in flight
}

}  // namespace ns
