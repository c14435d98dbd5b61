// batched.cuh -- the whole Newton step for a batch of independent paths of the
// same monomial structure, one CTA per path (persistent), every step of
// SURVEY 8(a) a1-a11 inside the CTA (independent units, no
// collective).  Warps evaluate/differentiate equations (warp-level
// convolutions, same reverse-mode job list as evaldiff.cuh); the QR of [A_0|I],
// the tile inversion and the stage loop use the CTA's shared memory.
#pragma once
#include "evaldiff.cuh"
#include "solve.cuh"

namespace ns {

// Byte offsets of the per-path arrays; each lives in shared memory when its
// `in_smem` bit is set, else in the CTA's global workspace slice.
struct BLayout {
  size_t off_W, off_invR, off_b, off_dx, off_y, off_vh, off_beta, off_kn;  // doubles
  unsigned in_smem;  // bit i for the arrays in the order above
  size_t smem_doubles;
  size_t gws_doubles;   // per CTA: A + per-warp series + arrays not in smem
  size_t off_A_g;       // in gws
  size_t off_ser_g;     // per-warp F/G/X series block in gws
};

template <int K>
__global__ void __launch_bounds__(256) batched_step_kernel(DevSys s, int batch, double* X, const double* RHS,
                                                           double* RES, double* gws_all, BLayout L,
                                                           int TB, long long* trace) {
  extern __shared__ double smem[];
  __shared__ int s_next;
  const int n = s.n, d = s.d, nnz = s.nnz;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, NW = blockDim.x >> 5;
  double* gws = gws_all + (size_t)blockIdx.x * L.gws_doubles;
  auto P = [&](int bit, size_t off) -> double* {
    return ((L.in_smem >> bit) & 1u) ? (smem + off) : (gws + off);
  };
  double* W = P(0, L.off_W);
  double* invR = P(1, L.off_invR);
  double* bb = P(2, L.off_b);    // b, then b' in place  [K][d][n]
  double* dxv = P(3, L.off_dx);  // [K][d][n]
  double* yv = P(4, L.off_y);    // [K][n]
  double* vh = P(5, L.off_vh);
  double* be = P(6, L.off_beta);
  double* kn = P(7, L.off_kn);   // [3][K][d]
  double* A = gws + L.off_A_g;   // [K][d][nnz]
  const long long ser = (long long)K * d;
  double* Fw = gws + L.off_ser_g + (size_t)warp * 3 * s.m_max * ser;
  double* Gw = Fw + s.m_max * ser;
  double* Xw = Gw + s.m_max * ser;
  const int ncol = 2 * n;
  const long long lsW = (long long)ncol * n, lsV = (long long)d * n, lsA = (long long)d * nnz;
  const long long lsX = (long long)n * d;
  const int T = (n + TB - 1) / TB;
  const long long lsI = (long long)T * TB * TB;

  // phase stamps (globaltimer) of the CTA's first path: start, eval/diff, QR, tiles, stages, residual
  long long* tr = (trace && tid == 0) ? trace + 8LL * blockIdx.x : nullptr;
  for (int p = blockIdx.x; p < batch; p += gridDim.x) {
    if (p != (int)blockIdx.x) tr = nullptr;
    if (tr) tr[0] = gtimer();
    double* x = X + (size_t)p * K * n * d;
    const double* rhs = RHS ? RHS + (size_t)p * K * n * d : s.rhs;
    // identity half of [A0 | I]
    for (long long t = tid; t < (long long)K * n * n; t += blockDim.x) {
      const int r = (int)(t % n);
      const long long lc = t / n;
      const int c = (int)(lc % n), l = (int)(lc / n);
      W[(long long)l * lsW + (long long)(n + c) * n + r] = (l == 0 && r == c) ? 1.0 : 0.0;
    }
    if (tid == 0) s_next = 0;
    __syncthreads();
    // ------------------------------------------------ eval/diff, warp per equation
    for (;;) {
      int job = 0;
      if (lane == 0) job = atomicAdd(&s_next, 1);
      job = __shfl_sync(0xffffffffu, job, 0);
      if (job >= n) break;
      const int i = s.job_order[job];
      const int r0 = s.row_ptr[i], len = s.row_ptr[i + 1] - r0;
      for (int t = lane; t < K * d; t += 32) {
        const int l = t / d, k = t % d;
        bb[(long long)l * lsV + (long long)k * n + i] = rhs[(long long)l * lsX + (long long)i * d + k];
      }
      for (int t = lane; t < K * d * len; t += 32) A[(long long)(t / len) * nnz + r0 + t % len] = 0.0;
      __syncwarp();
      for (int tau = s.eq_ptr[i]; tau < s.eq_ptr[i + 1]; ++tau) {
        const int m0 = s.mono_ptr[tau];
        const int m = s.mono_ptr[tau + 1] - m0;
        const int* vars = s.var_idx + m0;
        const int* dst = s.mono_dst + m0;
        md::mdv<K> c;
#pragma unroll
        for (int l = 0; l < K; ++l) c.x[l] = s.coeff[(long long)l * s.M + tau];
        if (m >= 2) {
          for (int q = 1; q <= m - 1; ++q) {
            const int nb = (q <= m - 2) ? 2 : 1;
            conv_batch<K>(lane, 32, nb, d, [&](int bi, SerRef& pa, SerRef& pb, double*& pc) {
              if (bi == 0) {
                pa = (q == 1) ? SerRef{x + (long long)vars[0] * d, lsX} : SerRef{Fw + (q - 1) * ser, d};
                pb = SerRef{x + (long long)vars[q] * d, lsX};
                pc = Fw + q * ser;
              } else {
                pa = (q == 1) ? SerRef{x + (long long)vars[m - 1] * d, lsX} : SerRef{Gw + (q - 1) * ser, d};
                pb = SerRef{x + (long long)vars[m - 1 - q] * d, lsX};
                pc = Gw + q * ser;
              }
            });
            __syncwarp();
          }
          if (m >= 3) {
            conv_batch<K>(lane, 32, m - 2, d, [&](int bi, SerRef& pa, SerRef& pb, double*& pc) {
              const int j = bi + 2;  // 1-based variable position
              pa = (j - 2 == 0) ? SerRef{x + (long long)vars[0] * d, lsX} : SerRef{Fw + (j - 2) * ser, d};
              const int gq = m - j - 1;
              pb = (gq == 0) ? SerRef{x + (long long)vars[m - 1] * d, lsX} : SerRef{Gw + gq * ser, d};
              pc = Xw + (j - 1) * ser;
            });
            __syncwarp();
          }
        }
        for (int k = lane; k < d; k += 32) {
          md::mdv<K> val = (m == 1) ? md::load<K>(x + (long long)vars[0] * d, lsX, k)
                                    : md::load<K>(Fw + (m - 1) * ser, d, k);
          md::mdv<K> acc = md::load<K>(bb + (long long)k * n, lsV, i);
          md::store<K>(bb + (long long)k * n, lsV, i, md::fma_acc<K>(acc, md::neg<K>(c), val));
        }
        for (int t = lane; t < m * d; t += 32) {
          const int q = t % m, k = t / m;
          md::mdv<K> part;
          if (m == 1) part = md::from_double<K>(k == 0 ? 1.0 : 0.0);
          else if (m == 2) part = md::load<K>(x + (long long)vars[1 - q] * d, lsX, k);
          else if (q == 0) part = md::load<K>(Gw + (m - 2) * ser, d, k);
          else if (q == m - 1) part = md::load<K>(Fw + (m - 2) * ser, d, k);
          else part = md::load<K>(Xw + q * ser, d, k);
          const long long e = dst[q];
          md::mdv<K> acc = md::load<K>(A + (long long)k * nnz, lsA, e);
          md::store<K>(A + (long long)k * nnz, lsA, e, md::fma_acc<K>(acc, c, part));
        }
        __syncwarp();
      }
      // dense row i of A0 into W (column-major): W[j][i]
      for (int t = lane; t < K * n; t += 32) {
        const int l = t / n, j = t % n;
        W[(long long)l * lsW + (long long)j * n + i] = 0.0;
      }
      __syncwarp();
      for (int t = lane; t < K * len; t += 32) {
        const int l = t / len, e = r0 + t % len;
        W[(long long)l * lsW + (long long)s.col_idx[e] * n + i] = A[(long long)l * lsA + e];
      }
      __syncwarp();
    }
    __syncthreads();
    if (tr) tr[1] = gtimer();
    // ||b_k||_1 of the evaluated b (before the stage loop turns b into b')
    for (int k = warp; k < d; k += NW) {
      md::mdv<K> acc = md::zero<K>();
      for (int i = lane; i < n; i += 32) acc = md::add<K>(acc, md::absv<K>(md::load<K>(bb + (long long)k * n, lsV, i)));
      acc = md::group_sum<K>(acc, 32);
      if (lane == 0) md::store<K>(kn, d, k, acc);
    }
    // ------------------------------------------------ Householder QR of [A0 | I]
    for (int j = 0; j < n; ++j) {
      if (warp == 0) make_reflector<K, false>(n, j, W, vh, be, nullptr, nullptr);
      __syncthreads();
      for (int c = j + 1 + warp; c < ncol; c += NW) apply_reflector<K, false>(n, j, c, W, vh, be);
      __syncthreads();
    }
    if (tr) tr[2] = gtimer();
    // ------------------------------------------------ inverses of R's diagonal tiles
    for (int tc = warp; tc < T * TB; tc += NW) {
      const int t = tc / TB, cl = tc % TB, t0 = t * TB;
      const int nb = min(TB, n - t0);
      md::mdv<K> inv_d = md::zero<K>();
      if (lane < nb) {
        md::mdv<K> rqq = md::load<K>(W, lsW, (long long)(t0 + lane) * n + t0 + lane);
        inv_d = md::recip<K>(rqq);
      }
      md::mdv<K> Xc = md::zero<K>();
      if (cl < nb) {
        if (lane == cl) Xc = inv_d;
        for (int r = cl - 1; r >= 0; --r) {
          md::mdv<K> pr = md::zero<K>();
          if (lane > r && lane <= cl)
            pr = md::mul<K>(md::load<K>(W, lsW, (long long)(t0 + lane) * n + t0 + r), Xc);
          pr = md::group_sum<K>(pr, 32);
          md::mdv<K> xr = md::neg<K>(md::mul<K>(pr, md::shfl<K>(inv_d, r)));
          if (lane == r) Xc = xr;
        }
      }
      if (lane < TB) {
        md::mdv<K> v = (lane < nb && cl < nb && lane <= cl) ? Xc : md::zero<K>();
        md::store<K>(invR, lsI, (long long)t * TB * TB + (long long)lane * TB + cl, v);
      }
    }
    __syncthreads();
    if (tr) tr[3] = gtimer();
    // ------------------------------------------------ stage loop
    for (int k = 0; k < d; ++k) {
      // updates: b'_k,i = b_k,i - sum_{j=1}^{k} sum_e A_j[e] dx_{k-j}[col e]
      if (k > 0) {
        for (int i = warp; i < n; i += NW) {
          const int r0 = s.row_ptr[i], len = s.row_ptr[i + 1] - r0;
          md::mdv<K> acc = md::zero<K>();
          for (int t = lane; t < k * len; t += 32) {
            const int j = 1 + t / len, e = r0 + t % len;
            acc = md::fma_acc<K>(acc, md::load<K>(A + (long long)j * nnz, lsA, e),
                                 md::load<K>(dxv + (long long)(k - j) * n, lsV, s.col_idx[e]));
          }
          acc = md::group_sum<K>(acc, 32);
          if (lane == 0) {
            md::mdv<K> bk = md::load<K>(bb + (long long)k * n, lsV, i);
            md::store<K>(bb + (long long)k * n, lsV, i, md::sub<K>(bk, acc));
          }
        }
        __syncthreads();
      }
      // qhb: y_r = sum_c (Q^T)[r][c] b'_k[c], Q^T in W columns n..2n-1 (thread per row)
      for (int r = tid; r < n; r += blockDim.x) {
        md::mdv<K> acc = md::zero<K>();
        for (int c = 0; c < n; ++c)
          acc = md::fma_acc<K>(acc, md::load<K>(W, lsW, (long long)(n + c) * n + r),
                               md::load<K>(bb + (long long)k * n, lsV, c));
        md::store<K>(yv, n, r, acc);
      }
      __syncthreads();
      // bs by tiles, last to first
      for (int t = T - 1; t >= 0; --t) {
        const int t0 = t * TB, t1 = min(n, t0 + TB);
        if (t < T - 1) {
          for (int r = t0 + tid; r < t1; r += blockDim.x) {
            md::mdv<K> acc = md::zero<K>();
            for (int c = t1; c < n; ++c)
              acc = md::fma_acc<K>(acc, md::load<K>(W, lsW, (long long)c * n + r),
                                   md::load<K>(dxv + (long long)k * n, lsV, c));
            md::store<K>(yv, n, r, md::sub<K>(md::load<K>(yv, n, r), acc));
          }
          __syncthreads();
        }
        for (int r = t0 + tid; r < t1; r += blockDim.x) {
          md::mdv<K> acc = md::zero<K>();
          for (int c = t0; c < t1; ++c)
            acc = md::fma_acc<K>(acc, md::load<K>(invR, lsI, (long long)t * TB * TB + (long long)(r - t0) * TB + (c - t0)),
                                 md::load<K>(yv, n, c));
          md::store<K>(dxv + (long long)k * n, lsV, r, acc);
        }
        __syncthreads();
      }
    }
    if (tr) tr[4] = gtimer();
    // ------------------------------------------------ residual r_k = b'_k - A_0 dx_k, norms
    for (int k = warp; k < d; k += NW) {
      md::mdv<K> nr = md::zero<K>(), nx = md::zero<K>();
      for (int i = lane; i < n; i += 32) {
        const int r0 = s.row_ptr[i], r1 = s.row_ptr[i + 1];
        md::mdv<K> acc = md::zero<K>();
        for (int e = r0; e < r1; ++e)
          acc = md::fma_acc<K>(acc, md::load<K>(A, lsA, e), md::load<K>(dxv + (long long)k * n, lsV, s.col_idx[e]));
        md::mdv<K> bpk = md::load<K>(bb + (long long)k * n, lsV, i);
        nr = md::add<K>(nr, md::absv<K>(md::sub<K>(bpk, acc)));
        nx = md::add<K>(nx, md::absv<K>(md::load<K>(dxv + (long long)k * n, lsV, i)));
      }
      nr = md::group_sum<K>(nr, 32);
      nx = md::group_sum<K>(nx, 32);
      if (lane == 0) {
        md::store<K>(kn + (long long)K * d, d, k, nr);
        md::store<K>(kn + 2LL * K * d, d, k, nx);
      }
    }
    __syncthreads();
    // x += dx
    for (int t = tid; t < n * d; t += blockDim.x) {
      const int j = t / d, k = t % d;
      md::store<K>(x, lsX, t, md::add<K>(md::load<K>(x, lsX, t), md::load<K>(dxv + (long long)k * n, lsV, j)));
    }
    if (RES && warp == 0 && lane < 3) {
      md::mdv<K> best = md::zero<K>();
      for (int k = 0; k < d; ++k) {
        md::mdv<K> v = md::load<K>(kn + (long long)lane * K * d, d, k);
        if (md::greater<K>(v, best)) best = v;
      }
      md::store<K>(RES + (size_t)p * K * 3, 3, lane, best);
    }
    __syncthreads();
    if (tr) tr[5] = gtimer();
  }
}

}  // namespace ns
