// evaldiff.cuh -- evaluation and differentiation of a monomial system at a
// power-series vector by reverse-mode AD over truncated series convolutions
// (Eq.(12)-(13); Eq.(14)).
//
// One CTA per equation (persistent, LPT order).  For each monomial
// tau = x_{v1} ... x_{vm} of the equation:
//   forward  f_1 = x_{v1} * x_{v2},  f_q = f_{q-1} * x_{v(q+1)}      q = 1..m-1
//   backward g_1 = x_{vm} * x_{v(m-1)}, g_q = g_{q-1} * x_{v(m-q)}   q = 1..m-2
//   cross    d/dx_{vj} = f_{j-2} * g_{m-j-1}  (f_0 = x_{v1}, g_0 = x_{vm}),  j = 2..m-1
//   value = f_{m-1},  d/dx_{v1} = g_{m-2},  d/dx_{vm} = f_{m-2}
// 3m-5 convolutions; m = 1, 2 per reading R7.  Layer q computes f_q and g_q
// together (two independent convolutions), the m-2 cross products run as one
// batch.  Then b_i = r_i - sum_tau c_tau value_tau and
// A[i][v] += c_tau d/dx_v, in ascending monomial order (reading R20).
//
// Convolution mapping (no zero padding, reading R6): output coefficients are
// paired (k, d-1-k) so every pair has d+1 terms; a group of G lanes shares a
// pair, each lane sums every G-th term with the fused md accumulate, and the
// group is reduced by a fixed butterfly (deterministic).
#pragma once
#include "common.cuh"

namespace ns {

struct SerRef {
  const double* p;  // coefficient 0 of limb plane 0
  long long ls;     // limb-plane stride
  bool cg = false;  // written by another SM in this kernel: load through L2 (ld.global.cg)
};

// Batched truncated convolutions c_b = a_b * b_b (b = 0..B-1) by the threads
// tid = 0..T-1 (a whole CTA, or one warp with T = 32).  get(bi, a, b, c)
// returns the operands of convolution bi; outputs are compact series (limb
// stride d).  T must be a multiple of 32 or equal to 32.
// Conv tuning (EdJobs.conv_mode): bit 0 selects the per-term renormalising
// accumulate (fma_acc, the first implementation); the default keeps each
// lane's partial sums as unnormalised level arrays (md::dot_levels_insert: the
// product's levels enter with exact two_sums, no renormalisation per term),
// reduces them with the lazy butterfly and renormalises once.  min_terms:
// the group width G doubles while every lane keeps >= min_terms terms.
template <int K, typename Get>
__device__ void conv_batch(int tid, int T, int B, int d, Get get, double* const* c2 = nullptr, int min_terms = 4,
                           int mode = 0, long long* dbg = nullptr, int ldc = 0) {
  // d: coefficients computed (the active window's dc); ldc: limb stride of the outputs (0: d)
  if (ldc == 0) ldc = d;
  const int P = (d + 1) / 2;
  const int groups = B * P;
  // G lanes per coefficient pair; each lane sums >= min_terms of the d+1 terms
  // (below that the md butterfly costs more than the multiply-adds)
  int G = 1;
  while (G < 32 && groups * G * 2 <= T && (d + 1) / (2 * G) >= min_terms) G <<= 1;
  const int per_round = T / G;
  const int sub = tid % G;
  for (int g0 = 0; g0 < groups; g0 += per_round) {
    const int gid = g0 + tid / G;
    const bool active = gid < groups;
    const int bi = active ? gid / P : 0;
    const int p = active ? gid % P : 0;
    const int k1 = p, k2 = d - 1 - p;
    const int tot = active ? ((k1 == k2) ? k1 + 1 : d + 1) : 0;
    SerRef a, b;
    double* c;
    get(bi, a, b, c);
    md::mdv<K> acc1, acc2;
    if (mode & 1) {
      acc1 = md::zero<K>();
      acc2 = md::zero<K>();
      for (int t = sub; t < tot; t += G) {
        const bool first = t <= k1;
        const int k = first ? k1 : k2;
        const int j = first ? t : t - k1 - 1;
        md::mdv<K> xa = a.cg ? md::load_cg<K>(a.p, a.ls, j) : md::load<K>(a.p, a.ls, j);
        md::mdv<K> yb = b.cg ? md::load_cg<K>(b.p, b.ls, k - j) : md::load<K>(b.p, b.ls, k - j);
        md::mdv<K> cur;
#pragma unroll
        for (int l = 0; l < K; ++l) cur.x[l] = first ? acc1.x[l] : acc2.x[l];
        cur = md::fma_acc<K>(cur, xa, yb);
#pragma unroll
        for (int l = 0; l < K; ++l) {
          acc1.x[l] = first ? cur.x[l] : acc1.x[l];
          acc2.x[l] = first ? acc2.x[l] : cur.x[l];
        }
      }
      if (G > 1) {
        acc1 = md::group_sum<K>(acc1, G);
        acc2 = md::group_sum<K>(acc2, G);
      }
    } else {
      // unnormalised level sums, UC terms per unrolled chunk (loads and
      // products of a chunk are independent; only the level inserts chain)
      constexpr int UC = (K <= 4) ? 4 : 2;
      double s1[K], s2[K];
#pragma unroll
      for (int l = 0; l < K; ++l) s1[l] = s2[l] = 0.0;
      // one term into the level sums of its output (first: k1, else k2)
      auto insert = [&](const md::mdv<K>& xa, const md::mdv<K>& yb, bool first) {
        double pl[K];
        md::prod_levels<K>(xa, yb, pl);
        double sc[K];
#pragma unroll
        for (int l = 0; l < K; ++l) sc[l] = first ? s1[l] : s2[l];
#pragma unroll
        for (int l = 0; l < K; ++l) md::level_insert<K>(sc, l, pl[l]);
#pragma unroll
        for (int l = 0; l < K; ++l) {
          s1[l] = first ? sc[l] : s1[l];
          s2[l] = first ? s2[l] : sc[l];
        }
      };
      auto operands = [&](int t, md::mdv<K>& xa, md::mdv<K>& yb, bool& first) {
        first = t <= k1;
        const int k = first ? k1 : k2;
        const int j = first ? t : t - k1 - 1;
        xa = a.cg ? md::load_cg<K>(a.p, a.ls, j) : md::load<K>(a.p, a.ls, j);
        yb = b.cg ? md::load_cg<K>(b.p, b.ls, k - j) : md::load<K>(b.p, b.ls, k - j);
      };
      int t0 = sub;
      for (; t0 + (UC - 1) * G < tot; t0 += UC * G) {  // full chunks
        md::mdv<K> xa[UC], yb[UC];
        bool fst[UC];
#pragma unroll
        for (int u = 0; u < UC; ++u) operands(t0 + u * G, xa[u], yb[u], fst[u]);
#pragma unroll
        for (int u = 0; u < UC; ++u) insert(xa[u], yb[u], fst[u]);
      }
      for (; t0 < tot; t0 += G) {  // tail terms
        md::mdv<K> xa, yb;
        bool first;
        operands(t0, xa, yb, first);
        insert(xa, yb, first);
      }
      if (dbg && tid == 0) dbg[0] = clock64();
      acc1 = md::group_sum_levels<K>(s1, G);
      acc2 = md::group_sum_levels<K>(s2, G);
      if (dbg && tid == 0) dbg[1] = clock64();
    }
    if (active && sub == 0) {
      md::store<K>(c, ldc, k1, acc1);
      if (k2 != k1) md::store<K>(c, ldc, k2, acc2);
      if (c2) {  // second copy (the chain's pool series next to its smem copy)
        md::store_cg<K>(c2[bi], ldc, k1, acc1);
        if (k2 != k1) md::store_cg<K>(c2[bi], ldc, k2, acc2);
      }
    }
  }
}

// ------------------------------------------------------------------ job-queue eval/diff
// Jobs (int4 {type, a, b, c}), popped in order by persistent CTAs:
//   JF  {0, tau}      forward chain f_1..f_{m-1} of monomial tau, publishes fprog[tau]
//   JG  {1, tau}      backward chain g_1..g_{m-2}, publishes gprog[tau]
//   JX  {2, tau, j}   cross product d/dx_{vj} = f_{j-2} * g_{m-j-1} (j = 2..m-1, 1-based)
//   JE  {3, i}        equation i: b_i = r_i - sum c value, A row, dense A0 row, in
//                     ascending monomial order (waits until its monomials are done)
// Every chain job precedes every cross job, which precede every equation job,
// so a job only ever waits for jobs popped earlier by resident CTAs: no
// deadlock.  Chains are ordered longest first (LPT), cross products by the
// layer at which their inputs appear.  Series live in a pool: F, G, X of
// monomial tau start at ser_off[tau] (compact [K][d] series, limb stride d).
struct EdJobs {
  const int4* jobs;
  int njobs;
  const long long* ser_off;  // [M] series index of f_1 of tau; g_1 at +m-1; d/dx_2 at +2m-3
  double* pool;
  int* fprog;                // [M] forward products done
  int* gprog;                // [M] backward products done
  int* left;                 // [M] chain + cross jobs not yet finished
  long long* trace;          // [njobs][3] pop / inputs-ready / done globaltimer (ns), or nullptr
  int conv_terms;            // conv_batch min_terms
  int conv_mode;             // conv_batch mode bits (bit 0: per-term renormalising accumulate;
                             // bit 1: cross jobs read their operands from the pool, no smem staging)
};

__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void wait_geq(const int* p, int v) {
  int ns = 32;
  while (ld_relaxed_s32(p) < v) {
    __nanosleep(ns);
    ns = min(ns * 2, 512);
  }
  (void)ld_acquire(p);
}
// asynchronous global -> shared copy of one double (cp.async, no register staging)
__device__ __forceinline__ void cp_async8(double* smem_dst, const double* gsrc) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_all;" ::: "memory");
}

// the CTA's pool writes are ordered before this by __syncthreads; the release
// store is cumulative (no separate fence)
__device__ __forceinline__ void publish(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int K>
__global__ void __launch_bounds__(256) evaldiff_jobs_kernel(DevSys s, EdJobs J, const double* __restrict__ x,
                                                            double* __restrict__ b, double* __restrict__ A,
                                                            double* __restrict__ A0, int* job_counter) {
  const int n = s.n, d = s.d, nnz = s.nnz;
  const long long ser = (long long)K * d;
  const long long xs = (long long)n * d;  // limb stride of x
  __shared__ int4 s_job;
  extern __shared__ double bacc[];  // [K][d]
  for (;;) {
    __shared__ int s_id;
    if (threadIdx.x == 0) {
      const int id = atomicAdd(job_counter, 1);
      s_job = (id < J.njobs) ? J.jobs[id] : make_int4(-1, 0, 0, 0);
      s_id = id;
      if (J.trace && id < J.njobs) J.trace[3LL * id] = gtimer();
    }
    __syncthreads();
    const int4 jb = s_job;
    __syncthreads();
    if (jb.x < 0) break;
    if (jb.x <= 2) {
      const int tau = jb.y;
      const int m0 = s.mono_ptr[tau];
      const int m = s.mono_ptr[tau + 1] - m0;
      const int* vars = s.var_idx + m0;
      double* F = J.pool + J.ser_off[tau] * ser;  // F[q-1] = f_q
      double* G = F + (m - 1) * ser;              // G[q-1] = g_q
      double* X = G + (m - 2) * ser;              // X[j-2] = d/dx_j
      if (jb.x <= 1) {
        // chain: forward (f_q = f_{q-1} * x_{v(q+1)}) or backward (g_q = g_{q-1} * x_{v(m-q)});
        // the running product stays in shared memory (double buffer), a copy goes
        // to the pool for the cross jobs and the equation job.
        const bool fwd = (jb.x == 0);
        const int len = fwd ? m - 1 : m - 2;
        double* base = fwd ? F : G;
        double* sbuf[2] = {bacc + K * d, bacc + 2 * K * d};
        double* xbuf[2] = {bacc + 3 * K * d, bacc + 4 * K * d};  // prefetched x series
        auto vidx = [&](int q) { return fwd ? vars[q] : vars[m - 1 - q]; };
        // x_{v(1)} (the first b operand) into xbuf[1]
        for (int t = threadIdx.x; t < K * d; t += blockDim.x) {
          const int l = t / d, k = t % d;
          cp_async8(&xbuf[1][l * d + k], x + (long long)l * xs + (long long)vidx(1) * d + k);
        }
        cp_async_wait_all();
        __syncthreads();
        long long* st_tr = (J.trace && s_id == 0) ? J.trace + 3LL * J.njobs : nullptr;  // step stamps of job 0
        for (int q = 1; q <= len; ++q) {
          if (st_tr && threadIdx.x == 0 && q <= 256) st_tr[4 * (q - 1)] = clock64();
          double* outp = base + (q - 1) * ser;
          // prefetch the next step's operand x_{v(q+1)} while this convolution runs
          if (q + 1 <= len)
            for (int t = threadIdx.x; t < K * d; t += blockDim.x) {
              const int l = t / d, k = t % d;
              cp_async8(&xbuf[(q + 1) & 1][l * d + k], x + (long long)l * xs + (long long)vidx(q + 1) * d + k);
            }
          auto get = [&](int, SerRef& pa, SerRef& pb, double*& pc) {
            pa = (q == 1) ? SerRef{x + (long long)vidx(0) * d, xs} : SerRef{sbuf[(q - 1) & 1], d};
            pb = SerRef{xbuf[q & 1], d};
            pc = sbuf[q & 1];
          };
          conv_batch<K>(threadIdx.x, blockDim.x, 1, s.dc, get, &outp, J.conv_terms, J.conv_mode,
                        (st_tr && q <= 256) ? st_tr + 4 * 256 + 2 * (q - 1) : nullptr, d);
          if (st_tr && threadIdx.x == 0 && q <= 256) st_tr[4 * (q - 1) + 1] = clock64();
          cp_async_wait_all();  // the next operand has landed (copy overlapped the convolution)
          __syncthreads();
          if (st_tr && threadIdx.x == 0 && q <= 256) st_tr[4 * (q - 1) + 2] = clock64();
          // the release store (a memory barrier) is issued by the last thread so that
          // warp 0, which computes, does not stall on it
          if (threadIdx.x == blockDim.x - 1) publish(fwd ? J.fprog + tau : J.gprog + tau, q);
        }
      } else {
        const int j = jb.z;  // 2..m-1
        if (threadIdx.x == 0) {
          if (j - 2 >= 1) wait_geq(J.fprog + tau, j - 2);
          if (m - j - 1 >= 1) wait_geq(J.gprog + tau, m - j - 1);
          if (J.trace) J.trace[3LL * s_id + 1] = gtimer();
        }
        __syncthreads();
        const int gq = m - j - 1;
        SerRef ra = (j - 2 == 0) ? SerRef{x + (long long)vars[0] * d, xs} : SerRef{F + (j - 3) * ser, d, true};
        SerRef rb = (gq == 0) ? SerRef{x + (long long)vars[m - 1] * d, xs} : SerRef{G + (gq - 1) * ser, d, true};
        if (!(J.conv_mode & 2)) {
          // both operands into shared memory (one L2 round trip instead of one per term chunk)
          double* sa = bacc + K * d;
          double* sb = bacc + 2 * K * d;
          for (int t = threadIdx.x; t < 2 * K * d; t += blockDim.x) {
            const int w = t / (K * d), r = t % (K * d);
            const int l = r / d, k = r % d;
            const SerRef& src = w ? rb : ra;
            cp_async8((w ? sb : sa) + l * d + k, src.p + l * src.ls + k);
          }
          cp_async_wait_all();
          __syncthreads();
          ra = SerRef{sa, d};
          rb = SerRef{sb, d};
        }
        auto get = [&](int, SerRef& pa, SerRef& pb, double*& pc) {
          pa = ra;
          pb = rb;
          pc = X + (j - 2) * ser;
        };
        conv_batch<K>(threadIdx.x, blockDim.x, 1, s.dc, get, nullptr, J.conv_terms, J.conv_mode, nullptr, d);
        __syncthreads();
      }
      if (threadIdx.x == 0) {
        __threadfence();
        atomicSub(J.left + tau, 1);
        if (J.trace) J.trace[3LL * s_id + 2] = gtimer();
      }
      continue;
    }
    // ---- JE: equation i
    const int i = jb.y;
    const int r0 = s.row_ptr[i], r1 = s.row_ptr[i + 1];
    if (threadIdx.x == 0)
      for (int tau = s.eq_ptr[i]; tau < s.eq_ptr[i + 1]; ++tau) {
        int ns = 32;
        while (ld_relaxed_s32(J.left + tau) > 0) {
          __nanosleep(ns);
          ns = min(ns * 2, 512);
        }
        (void)ld_acquire(J.left + tau);
      }
    if (threadIdx.x == 0 && J.trace) J.trace[3LL * s_id + 1] = gtimer();
    for (int t = threadIdx.x; t < K * d; t += blockDim.x) {
      const int l = t / d, k = t % d;
      bacc[l * d + k] = s.rhs[(long long)l * xs + (long long)i * d + k];
    }
    for (long long t = threadIdx.x; t < (long long)K * d * (r1 - r0); t += blockDim.x) {
      const int e = r0 + (int)(t % (r1 - r0));
      const long long lk = t / (r1 - r0);
      A[lk * nnz + e] = 0.0;
    }
    __syncthreads();
    for (int tau = s.eq_ptr[i]; tau < s.eq_ptr[i + 1]; ++tau) {
      const int m0 = s.mono_ptr[tau];
      const int m = s.mono_ptr[tau + 1] - m0;
      const int* vars = s.var_idx + m0;
      const int* dst = s.mono_dst + m0;
      const double* F = J.pool + J.ser_off[tau] * ser;
      const double* G = F + (m - 1) * ser;
      const double* X = G + (m - 2) * ser;
      md::mdv<K> c;
#pragma unroll
      for (int l = 0; l < K; ++l) c.x[l] = s.coeff[(long long)l * s.M + tau];
      for (int k = threadIdx.x; k < s.dc; k += blockDim.x) {
        md::mdv<K> val = (m == 1) ? md::load<K>(x + (long long)vars[0] * d, xs, k)
                                  : md::load_cg<K>(F + (m - 2) * ser, d, k);
        md::mdv<K> acc = md::load<K>(bacc, d, k);
        md::store<K>(bacc, d, k, md::fma_acc<K>(acc, md::neg<K>(c), val));
      }
      // with repeated variables (exponent > 1) several occurrences q share an
      // entry: one thread per coefficient k then runs over q in order
      const int qs = s.repeats ? m : 1;
      for (int t = threadIdx.x; t < (m / qs) * s.dc; t += blockDim.x) {
        for (int qq = 0; qq < qs; ++qq) {
          const int q = s.repeats ? qq : t % m, k = s.repeats ? t : t / m;
          md::mdv<K> part;
          if (m == 1) part = md::from_double<K>(k == 0 ? 1.0 : 0.0);
          else if (m == 2) part = md::load<K>(x + (long long)vars[1 - q] * d, xs, k);
          else if (q == 0) part = md::load_cg<K>(G + (m - 3) * ser, d, k);        // g_{m-2}
          else if (q == m - 1) part = md::load_cg<K>(F + (m - 3) * ser, d, k);    // f_{m-2}
          else part = md::load_cg<K>(X + (q - 1) * ser, d, k);                    // d/dx_{q+1}
          const long long e = dst[q];
          md::mdv<K> acc = md::load<K>(A + (long long)k * nnz, (long long)d * nnz, e);
          md::store<K>(A + (long long)k * nnz, (long long)d * nnz, e, md::fma_acc<K>(acc, c, part));
        }
      }
      __syncthreads();
    }
    for (int t = threadIdx.x; t < K * d; t += blockDim.x) {
      const int l = t / d, k = t % d;
      b[((long long)l * d + k) * n + i] = bacc[l * d + k];
    }
    for (int t = threadIdx.x; t < K * n; t += blockDim.x) {
      const int l = t / n, j = t % n;
      A0[((long long)l * n + i) * n + j] = 0.0;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < K * (r1 - r0); t += blockDim.x) {
      const int l = t / (r1 - r0), e = r0 + t % (r1 - r0);
      A0[((long long)l * n + i) * n + s.col_idx[e]] = A[(long long)l * d * nnz + e];
    }
    __syncthreads();
    if (threadIdx.x == 0 && J.trace) J.trace[3LL * s_id + 2] = gtimer();
  }
}

}  // namespace ns

namespace ns {
// Dense A_0 alone (the t^0 coefficients of the Jacobian), for the QR to start
// before the full eval/diff finishes: A_0[i][v_q] = sum_tau c_tau prod_{r != q} x_{v_r,0}.
// One warp per equation; prefix and suffix products of the m scalars by a
// chunked warp scan (md multiplications in a fixed order), so the dependent
// chain is ~2 ceil(m/32) + 5 products instead of m.
template <int K>
__device__ md::mdv<K> warp_excl_scan_mul(md::mdv<K> v) {
  const int lane = threadIdx.x & 31;
  // inclusive Hillis-Steele scan, then shift by one
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    md::mdv<K> o = md::shfl<K>(v, max(lane - off, 0));
    if (lane >= off) v = md::mul<K>(o, v);
  }
  md::mdv<K> e = md::shfl<K>(v, max(lane - 1, 0));
  return lane == 0 ? md::from_double<K>(1.0) : e;
}

// Row i of A_0 into dst[(l * plane) + i * rs + j * cs] (row-major: rs = n, cs = 1;
// column-major W: rs = 1, cs = n), one warp.
template <int K>
__device__ void a0_row(const DevSys& s, const double* __restrict__ x, int i, double* dst, long long plane,
                       long long rs, long long cs) {
  const int n = s.n, d = s.d;
  const long long xs = (long long)n * d;
  const int lane = threadIdx.x & 31;
  for (int j = lane; j < n; j += 32) md::store<K>(dst, plane, i * rs + j * cs, md::zero<K>());
  __syncwarp();
  for (int tau = s.eq_ptr[i]; tau < s.eq_ptr[i + 1]; ++tau) {
    const int m0 = s.mono_ptr[tau], m = s.mono_ptr[tau + 1] - m0;
    const int* vars = s.var_idx + m0;
    md::mdv<K> c;
#pragma unroll
    for (int l = 0; l < K; ++l) c.x[l] = s.coeff[(long long)l * s.M + tau];
    const int C = (m + 31) / 32;  // chunk per lane
    const int q0 = lane * C;
    md::mdv<K> lp = md::from_double<K>(1.0), ls = md::from_double<K>(1.0);
    for (int q = q0; q < min(m, q0 + C); ++q) lp = md::mul<K>(lp, md::load<K>(x + (long long)vars[q] * d, xs, 0));
    for (int q = min(m, q0 + C) - 1; q >= q0; --q) ls = md::mul<K>(md::load<K>(x + (long long)vars[q] * d, xs, 0), ls);
    const md::mdv<K> pre = warp_excl_scan_mul<K>(lp);
    const md::mdv<K> rv = md::shfl<K>(ls, 31 - lane);
    const md::mdv<K> sufr = warp_excl_scan_mul<K>(rv);
    const md::mdv<K> suf = md::shfl<K>(sufr, 31 - lane);
    md::mdv<K> P = pre;
    // repeated variables (exponent > 1) share an entry across lanes: the lanes
    // then add their occurrences in lane order (one lane at a time)
    for (int L = 0; L < (s.repeats ? 32 : 1); ++L) {
      if (!s.repeats || lane == L)
        for (int q = q0; q < min(m, q0 + C); ++q) {
          md::mdv<K> S = suf;
          for (int r = min(m, q0 + C) - 1; r > q; --r) S = md::mul<K>(md::load<K>(x + (long long)vars[r] * d, xs, 0), S);
          const md::mdv<K> part = md::mul<K>(P, S);
          const long long e = i * rs + (long long)vars[q] * cs;
          md::store<K>(dst, plane, e, md::fma_acc<K>(md::load<K>(dst, plane, e), c, part));
          P = md::mul<K>(P, md::load<K>(x + (long long)vars[q] * d, xs, 0));
        }
      __syncwarp();
    }
  }
}

template <int K>
__global__ void __launch_bounds__(128) a0_kernel(DevSys s, const double* __restrict__ x, double* __restrict__ A0q) {
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int i = gw; i < s.n; i += nw) a0_row<K>(s, x, i, A0q, (long long)s.n * s.n, s.n, 1);
}
}  // namespace ns
