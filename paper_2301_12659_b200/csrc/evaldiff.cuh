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
};

// Batched truncated convolutions c_b = a_b * b_b (b = 0..B-1) by the threads
// tid = 0..T-1 (a whole CTA, or one warp with T = 32).  get(bi, a, b, c)
// returns the operands of convolution bi; outputs are compact series (limb
// stride d).  T must be a multiple of 32 or equal to 32.
template <int K, typename Get>
__device__ void conv_batch(int tid, int T, int B, int d, Get get) {
  const int P = (d + 1) / 2;
  const int groups = B * P;
  int G = 1;
  while (G < 32 && groups * G * 2 <= T) G <<= 1;
  const int per_round = T / G;
  const int sub = tid % G;
  for (int g0 = 0; g0 < groups; g0 += per_round) {
    const int gid = g0 + tid / G;
    const bool active = gid < groups;
    const int bi = active ? gid / P : 0;
    const int p = active ? gid % P : 0;
    const int k1 = p, k2 = d - 1 - p;
    const int tot = active ? ((k1 == k2) ? k1 + 1 : d + 1) : 0;
    md::mdv<K> acc1 = md::zero<K>(), acc2 = md::zero<K>();
    SerRef a, b;
    double* c;
    get(bi, a, b, c);
    for (int t = sub; t < tot; t += G) {
      const bool first = t <= k1;
      const int k = first ? k1 : k2;
      const int j = first ? t : t - k1 - 1;
      md::mdv<K> x = md::load<K>(a.p, a.ls, j);
      md::mdv<K> y = md::load<K>(b.p, b.ls, k - j);
      md::mdv<K> cur;
#pragma unroll
      for (int l = 0; l < K; ++l) cur.x[l] = first ? acc1.x[l] : acc2.x[l];
      cur = md::fma_acc<K>(cur, x, y);
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
    if (active && sub == 0) {
      md::store<K>(c, d, k1, acc1);
      if (k2 != k1) md::store<K>(c, d, k2, acc2);
    }
  }
}

// Per-CTA workspace: F[m_max], G[m_max], X[m_max] compact series (K*d doubles each)
template <int K>
__global__ void __launch_bounds__(256) evaldiff_kernel(DevSys s, const double* __restrict__ x,
                                                       double* __restrict__ b, double* __restrict__ A,
                                                       double* __restrict__ A0, double* __restrict__ ws,
                                                       int* job_counter) {
  const int n = s.n, d = s.d, nnz = s.nnz;
  const long long ser = (long long)K * d;
  double* F = ws + (long long)blockIdx.x * 3 * s.m_max * ser;
  double* Gs = F + s.m_max * ser;
  double* X = Gs + s.m_max * ser;
  __shared__ SerRef sa[64], sb[64];
  __shared__ double* sc[64];
  __shared__ int s_job;
  extern __shared__ double bacc[];  // [K][d]

  const long long xs = (long long)n * d;  // limb stride of x
  for (;;) {
    if (threadIdx.x == 0) s_job = atomicAdd(job_counter, 1);
    __syncthreads();
    const int job = s_job;
    __syncthreads();
    if (job >= n) break;
    const int i = s.job_order[job];
    const int r0 = s.row_ptr[i], r1 = s.row_ptr[i + 1];
    // b accumulator starts at r_i(t); zero the structural row of A
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
      md::mdv<K> c;
#pragma unroll
      for (int l = 0; l < K; ++l) c.x[l] = s.coeff[(long long)l * s.M + tau];
      // ---- forward / backward chains (layers) and cross products
      if (m >= 2) {
        for (int q = 1; q <= m - 1; ++q) {
          if (threadIdx.x == 0) {
            int nb = 0;
            sa[nb] = (q == 1) ? SerRef{x + (long long)vars[0] * d, xs} : SerRef{F + (q - 1) * ser, d};
            sb[nb] = SerRef{x + (long long)vars[q] * d, xs};
            sc[nb] = F + q * ser;
            ++nb;
            if (q <= m - 2) {
              sa[nb] = (q == 1) ? SerRef{x + (long long)vars[m - 1] * d, xs} : SerRef{Gs + (q - 1) * ser, d};
              sb[nb] = SerRef{x + (long long)vars[m - 1 - q] * d, xs};
              sc[nb] = Gs + q * ser;
              ++nb;
            }
            s_job = nb;
          }
          __syncthreads();
          const int nb = s_job;
          conv_batch<K>(threadIdx.x, blockDim.x, nb, d, [&](int bi, SerRef& pa, SerRef& pb, double*& pc) {
            pa = sa[bi]; pb = sb[bi]; pc = sc[bi];
          });
          __syncthreads();
        }
        // cross products d/dx_{vj}, j = 2..m-1 (1-based) -> X[j-1]
        for (int j0 = 2; j0 <= m - 1; j0 += 64) {
          const int cnt = min(64, m - j0);
          if (threadIdx.x < cnt) {
            const int j = j0 + threadIdx.x;
            sa[threadIdx.x] = (j - 2 == 0) ? SerRef{x + (long long)vars[0] * d, xs} : SerRef{F + (j - 2) * ser, d};
            const int gq = m - j - 1;
            sb[threadIdx.x] = (gq == 0) ? SerRef{x + (long long)vars[m - 1] * d, xs} : SerRef{Gs + gq * ser, d};
            sc[threadIdx.x] = X + (j - 1) * ser;
          }
          __syncthreads();
          conv_batch<K>(threadIdx.x, blockDim.x, cnt, d, [&](int bi, SerRef& pa, SerRef& pb, double*& pc) {
            pa = sa[bi]; pb = sb[bi]; pc = sc[bi];
          });
          __syncthreads();
        }
      }
      // ---- b_i -= c * value ; A[i][v_q] += c * d/dx_{v_q}
      for (int k = threadIdx.x; k < d; k += blockDim.x) {
        md::mdv<K> val;
        if (m == 1) val = md::load<K>(x + (long long)vars[0] * d, xs, k);
        else val = md::load<K>(F + (m - 1) * ser, d, k);
        md::mdv<K> acc = md::load<K>(bacc, d, k);
        acc = md::fma_acc<K>(acc, md::neg<K>(c), val);
        md::store<K>(bacc, d, k, acc);
      }
      for (int t = threadIdx.x; t < m * d; t += blockDim.x) {
        const int q = t % m, k = t / m;
        md::mdv<K> part;
        if (m == 1) {
          part = md::from_double<K>(k == 0 ? 1.0 : 0.0);
        } else if (m == 2) {
          part = md::load<K>(x + (long long)vars[1 - q] * d, xs, k);
        } else if (q == 0) {
          part = md::load<K>(Gs + (m - 2) * ser, d, k);
        } else if (q == m - 1) {
          part = md::load<K>(F + (m - 2) * ser, d, k);
        } else {
          part = md::load<K>(X + q * ser, d, k);
        }
        const long long e = dst[q];
        md::mdv<K> acc = md::load<K>(A + (long long)k * nnz, (long long)d * nnz, e);
        acc = md::fma_acc<K>(acc, c, part);
        md::store<K>(A + (long long)k * nnz, (long long)d * nnz, e, acc);
      }
      __syncthreads();
    }
    // ---- write b column i and the dense row i of A0
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
  }
}

}  // namespace ns
