// batched.cuh -- the whole Newton step for a batch of
// independent paths of one monomial structure, one CTA per path (persistent;
// independent units, no collective), real or complex scalars
// (scalar.cuh; NEXT-2).
//
// Per path, inside the CTA (arrays in shared memory when the layout fits,
// else in the CTA's slice of the global workspace, BLayout):
//   eval/diff   warp per equation (LPT order), reverse mode of Eq.(12): the
//               forward and backward chains of a monomial advance together,
//               the cross products run as one batch; every convolution output
//               pair (k, d-1-k) is summed by ONE lane (d+1 terms, no padding,
//               no butterfly), the accumulation in unnormalised level sums
//               renormalised once per output.  b_i = r_i - sum c x^tau and the
//               A row in ascending monomial order (reading R20).
//   QR          Householder on [A_0 | I]: a group of TPC lanes owns a
//               column (rows dealt round robin), reflector j by the group of
//               column j, then every other column group applies it; after n
//               steps W = [R | Q^H].  Complex: alpha = -(x_0/|x_0|) ||x||,
//               beta = 1 / (||x|| (||x|| + |x_0|)) (reading R13 generalised).
//   tiles       inverses of the TB x TB diagonal tiles of R (recursive doubling)
//   stages      for k = 0..D: y = Q^H b'_k, tiled back substitution
//               R dx_k = y, then right-looking updates
//               b'_{k'} -= A_{k'-k} dx_k for every k' > k (the updates of
//               P:680-689 applied as soon as dx_k exists; per (k', i) the
//               contributions k = 0, 1, ... arrive in order: deterministic)
//   residual    r_k = b'_k - A_0 dx_k, norms, x += dx.
// Only __syncthreads between phases; no grid-wide synchronisation.
#pragma once
#include "evaldiff.cuh"
#include "scalar.cuh"
#include "system.h"

namespace ns {

// BLayout and the array ids B_* are in system.h (the host sizes the layout)

template <class A>
MD_INL void acc_select(A& dst, const A& x, const A& y, bool take_x) {
  constexpr int N = sizeof(A) / sizeof(double);
  double* o = reinterpret_cast<double*>(&dst);
  const double* a = reinterpret_cast<const double*>(&x);
  const double* b = reinterpret_cast<const double*>(&y);
#pragma unroll
  for (int i = 0; i < N; ++i) o[i] = take_x ? a[i] : b[i];
}

struct BSer {
  const double* p;  // coefficient 0 of limb plane 0 of component 0
  long long ls;     // limb-plane stride
};

// B truncated convolutions out_b = a_b * b_b (b < B; get() returns false for
// an inactive item) on one warp: lane per
// output pair (k1, k2 = d-1-k1), both sums in one loop of d+1 terms (k1 + 1
// terms of c_{k1}, then k2 + 1 of c_{k2}) with the accumulator chosen per
// term (no divergence), outputs compact series (limb stride ldo).
// the same with the outputs handed to emit(bi, out, k, value) (an epilogue)
template <class S, typename Get, typename Emit>
__device__ __forceinline__ void sconv_warp_emit(int lane, int B, int d, Get get, Emit emit) {
  using V = typename S::V;
  using Acc = typename S::Acc;
  const int P = (d + 1) / 2;
  for (int g0 = 0; g0 < B * P; g0 += 32) {
    const int gid = g0 + lane;
    if (gid < B * P) {
      const int bi = gid / P, p = gid % P;
      const int k1 = p, k2 = d - 1 - p;
      const int tot = (k1 == k2) ? k1 + 1 : d + 1;
      BSer a, b;
      double* out;
      if (get(bi, a, b, out)) {
      Acc a1, a2;
      S::acc_zero(a1);
      S::acc_zero(a2);
      for (int t = 0; t < tot; ++t) {
        const bool first = t <= k1;
        const int k = first ? k1 : k2;
        const int j = first ? t : t - k1 - 1;
        const V xa = S::load(a.p, a.ls, j), yb = S::load(b.p, b.ls, k - j);
        Acc cur;
        acc_select(cur, a1, a2, first);
        S::acc_prod(cur, xa, yb);
        acc_select(a1, cur, a1, first);
        acc_select(a2, a2, cur, first);
      }
      emit(bi, out, k1, S::val(a1));
      if (k2 != k1) emit(bi, out, k2, S::val(a2));
      }
    }
  }
}

template <class S, typename Get>
__device__ __forceinline__ void sconv_warp(int lane, int B, int d, int ldo, Get get) {
  sconv_warp_emit<S>(lane, B, d, get, [&](int, double* out, int k, const typename S::V& v) { S::store(out, ldo, k, v); });
}


// MB: minimum CTAs per SM the register allocation must allow (launch bounds)
template <class S, int K, int MB>
__global__ void __launch_bounds__(256, MB) batched_step_kernel(DevSys s, int batch, double* X, const double* RHS,
                                                           double* RES, double* gws_all, BLayout L,
                                                           long long* trace) {
  using V = typename S::V;
  using R = typename S::R;
  using Acc = typename S::Acc;
  constexpr int C = S::C;
  extern __shared__ double smem[];
  __shared__ int s_next;
  const int n = s.n, d = s.d, nnz = s.nnz;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, NT = blockDim.x;
  double* gws = gws_all + (size_t)blockIdx.x * L.gws_doubles;
  auto Pa = [&](int a) -> double* { return ((L.in_smem >> a) & 1u) ? (smem + L.off[a]) : (gws + L.off[a]); };
  double* xs = Pa(B_X);    // x    [C][K][n][d]
  double* bb = Pa(B_B);    // b -> pending b' -> r  [C][K][d][n]
  double* dxv = Pa(B_DX);  // dx   [C][K][d][n]
  double* W = Pa(B_W);     // [A_0 | I] -> [R | Q^H], column major [C][K][2n][n]
  double* RI = Pa(B_RI);   // inverted diagonal tiles of R [C][K][T][TB][TB]
  double* yv = Pa(B_Y);    // y = Q^H b'_k, scratch of the tile inverses [C][K][max(n, TB^2/2)]
  double* vh = Pa(B_VH);   // v_0 of each reflector [C][K][n]
  double* be = Pa(B_BE);   // beta of each reflector (real) [K][n]
  double* kn = Pa(B_KN);   // per-k norms (real) [3][K][d]: b, r, dx
  double* A = gws + L.off_A_g;  // [C][K][d][nnz]
  const long long lsX = (long long)n * d, lsV = (long long)d * n, lsW = 2LL * n * n, lsA = (long long)d * nnz;
  const int TB = L.TB, T = (n + TB - 1) / TB, TT = TB * TB;
  const long long lsI = (long long)T * TT;
  const long long lsY = (long long)max(n, TT / 2);
  const long long ser = (long long)C * K * d;  // one compact series
  double* Fw = gws + L.off_ser_g + (size_t)warp * 2 * 3 * s.m_max * ser;  // two equations: [2][F, G, X]
  const int ncol = 2 * n;
  int TPC = 1;  // lanes per column of the QR (power of two <= 32, ncol TPC <= NT)
  while (TPC < 32 && ncol * TPC * 2 <= NT) TPC <<= 1;
  int TPO = 1;  // lanes per output of the Q^H and tile matvecs
  while (TPO < 32 && n * TPO * 2 <= NT) TPO <<= 1;
  long long* tr = (trace && tid == 0) ? trace + 8LL * blockIdx.x : nullptr;

  for (int p = blockIdx.x; p < batch; p += gridDim.x) {
    if (p != (int)blockIdx.x) tr = nullptr;
    if (tr) tr[0] = gtimer();
    double* xg = X + (size_t)p * C * K * n * d;
    const double* rhs = RHS ? RHS + (size_t)p * C * K * n * d : s.rhs;
    // ---------------------------------------------------- inputs: x, b = r, I half of W
    for (int t = tid; t < C * K * n * d; t += NT) {
      xs[t] = xg[t];
      const int ck = t / (n * d), r = t % (n * d), i = r / d, k = r % d;
      bb[(long long)ck * lsV + (long long)k * n + i] = rhs[t];
    }
    for (long long t = tid; t < (long long)C * K * n * n; t += NT) {
      const int r = (int)(t % n);
      const long long lc = t / n;
      const int c = (int)(lc % n), ck = (int)(lc / n);
      W[(long long)ck * lsW + (long long)(n + c) * n + r] = (ck == 0 && r == c) ? 1.0 : 0.0;
    }
    if (tid == 0) s_next = 0;
    __syncthreads();
    // ---------------------------------------------------- eval/diff, warp per pair of equations
    // Two equations (consecutive in the LPT order, so of similar cost) advance
    // in lockstep: their u-th monomials' forward and backward chains share
    // each layer's convolution batch (up to 4 series x (d+1)/2 output pairs
    // on the 32 lanes) and their cross products one batch, so the chain layers
    // do not leave half of the warp idle.  Each equation keeps its own
    // series (F, G, X per slot) and its own ascending monomial order.
    for (;;) {
      int job = 0;
      if (lane == 0) job = atomicAdd(&s_next, 1);
      job = __shfl_sync(0xffffffffu, job, 0);
      if (2 * job >= n) break;
      const int eqs0 = s.job_order[2 * job];
      const int eqs1 = (2 * job + 1 < n) ? s.job_order[2 * job + 1] : -1;
      for (int e2 = 0; e2 < 2; ++e2) {
        const int i = e2 ? eqs1 : eqs0;
        if (i < 0) continue;
        const int r0 = s.row_ptr[i], len = s.row_ptr[i + 1] - r0;
        for (int t = lane; t < C * K * d * len; t += 32) A[(long long)(t / len) * nnz + r0 + t % len] = 0.0;
      }
      __syncwarp();
      const int nmono0 = s.eq_ptr[eqs0 + 1] - s.eq_ptr[eqs0];
      const int nmono1 = (eqs1 >= 0) ? s.eq_ptr[eqs1 + 1] - s.eq_ptr[eqs1] : 0;
      for (int u = 0; u < max(nmono0, nmono1); ++u) {
        // the u-th monomial of each equation of the pair (m = 0: none); scalars
        // selected by e2 (no dynamically indexed local arrays)
        const int tau0 = (u < nmono0) ? s.eq_ptr[eqs0] + u : -1;
        const int tau1 = (u < nmono1) ? s.eq_ptr[eqs1] + u : -1;
        const int m0_ = (tau0 >= 0) ? s.mono_ptr[tau0 + 1] - s.mono_ptr[tau0] : 0;
        const int m1_ = (tau1 >= 0) ? s.mono_ptr[tau1 + 1] - s.mono_ptr[tau1] : 0;
        const int* vv0 = s.var_idx + ((tau0 >= 0) ? s.mono_ptr[tau0] : 0);
        const int* vv1 = s.var_idx + ((tau1 >= 0) ? s.mono_ptr[tau1] : 0);
        auto TAU = [&](int e2) { return e2 ? tau1 : tau0; };
        auto MM = [&](int e2) { return e2 ? m1_ : m0_; };
        auto VV = [&](int e2) { return e2 ? vv1 : vv0; };
        auto xser = [&](int v) { return BSer{xs + (long long)v * d, lsX}; };
        const int layers = max(m0_, m1_) - 1;
        // layer q: f_q = f_{q-1} * x_{v(q+1)} and g_q = g_{q-1} * x_{v(m-q)} (Eq.(12))
        for (int q = 1; q <= layers; ++q) {
          sconv_warp<S>(lane, 4, d, d, [&](int bi, BSer& pa, BSer& pb, double*& pc) -> bool {
            const int e2 = bi >> 1, m = MM(e2);
            const int* vars = VV(e2);
            double* F = Fw + (size_t)e2 * 3 * s.m_max * ser;
            double* G = F + s.m_max * ser;
            if ((bi & 1) == 0) {
              if (q > m - 1) return false;
              pa = (q == 1) ? xser(vars[0]) : BSer{F + (q - 1) * ser, d};
              pb = xser(vars[q]);
              pc = F + q * ser;
            } else {
              if (q > m - 2) return false;
              pa = (q == 1) ? xser(vars[m - 1]) : BSer{G + (q - 1) * ser, d};
              pb = xser(vars[m - 1 - q]);
              pc = G + q * ser;
            }
            return true;
          });
          __syncwarp();
        }
        // cross products d/dx_{v_j} = f_{j-2} * g_{m-j-1}, j = 2..m-1 (Eq.(13)), both equations
        const int nx0 = max(0, m0_ - 2), nx1 = max(0, m1_ - 2);
        // without repeated variables every interior partial (occurrence q = j-1,
        // 1 <= q <= m-2) has its own A entry: the convolution's epilogue adds
        // c d/dx_{v_j} x^tau into A directly (no X series round trip); the
        // boundary partials and m <= 2 follow below, still in monomial order
        const bool fuse = !s.repeats;
        auto emit_x = [&](int bi, double* out, int k, const V& v) {
          if (!fuse) {
            S::store(out, d, k, v);
            return;
          }
          const int e2 = (bi < nx0) ? 0 : 1;
          const int q = (bi < nx0 ? bi : bi - nx0) + 1;
          const long long e = s.mono_dst[s.mono_ptr[TAU(e2)] + q];
          const V c = S::load(s.coeff, s.M, TAU(e2));
          S::store(A + (long long)k * nnz, lsA, e, S::fma(S::load(A + (long long)k * nnz, lsA, e), c, v));
        };
        if (nx0 + nx1 > 0) {
          sconv_warp_emit<S>(lane, nx0 + nx1, d, [&](int bi, BSer& pa, BSer& pb, double*& pc) -> bool {
            const int e2 = (bi < nx0) ? 0 : 1, m = MM(e2);
            const int j = (bi < nx0 ? bi : bi - nx0) + 2;
            const int* vars = VV(e2);
            double* F = Fw + (size_t)e2 * 3 * s.m_max * ser;
            double* G = F + s.m_max * ser;
            double* X = G + s.m_max * ser;
            pa = (j - 2 == 0) ? xser(vars[0]) : BSer{F + (j - 2) * ser, d};
            const int gq = m - j - 1;
            pb = (gq == 0) ? xser(vars[m - 1]) : BSer{G + gq * ser, d};
            pc = X + (j - 1) * ser;
            return true;
          }, emit_x);
          __syncwarp();
        }
        for (int e2 = 0; e2 < 2; ++e2) {
          const int m = MM(e2);
          if (m == 0) continue;
          const int i = e2 ? eqs1 : eqs0;
          const int* vars = VV(e2);
          const int* dst = s.mono_dst + s.mono_ptr[TAU(e2)];
          const V c = S::load(s.coeff, s.M, TAU(e2));
          const double* F = Fw + (size_t)e2 * 3 * s.m_max * ser;
          const double* G = F + s.m_max * ser;
          const double* X = G + s.m_max * ser;
          for (int k = lane; k < d; k += 32) {  // b_i -= c x^tau
            const V val = (m == 1) ? S::load(xs + (long long)vars[0] * d, lsX, k) : S::load(F + (m - 1) * ser, d, k);
            S::store(bb + (long long)k * n, lsV, i, S::fma(S::load(bb + (long long)k * n, lsV, i), S::neg(c), val));
          }
          // A[i][v_q] += c d x^tau / d x_{v_q}; repeated variables (exponent > 1)
          // share an entry: a lane per coefficient then runs over q in order
          // fused: only the boundary occurrences q = 0, m-1 remain (m >= 3)
          const int mq = (fuse && m >= 3) ? 2 : m;
          for (int t = lane; t < (mq / (s.repeats ? mq : 1)) * d; t += 32) {
            for (int qq = 0; qq < (s.repeats ? mq : 1); ++qq) {
              const int q0 = s.repeats ? qq : t % mq, k = s.repeats ? t : t / mq;
              const int q = (mq == 2 && m >= 3) ? (q0 == 0 ? 0 : m - 1) : q0;
              V part;
              if (m == 1) part = (k == 0) ? S::one() : S::zero();
              else if (m == 2) part = S::load(xs + (long long)vars[1 - q] * d, lsX, k);
              else if (q == 0) part = S::load(G + (m - 2) * ser, d, k);
              else if (q == m - 1) part = S::load(F + (m - 2) * ser, d, k);
              else part = S::load(X + q * ser, d, k);
              const long long e = dst[q];
              S::store(A + (long long)k * nnz, lsA, e, S::fma(S::load(A + (long long)k * nnz, lsA, e), c, part));
            }
          }
        }
        __syncwarp();
      }
      // dense rows of A_0 into W (column major: W[j][i])
      for (int e2 = 0; e2 < 2; ++e2) {
        const int i = e2 ? eqs1 : eqs0;
        if (i < 0) continue;
        const int r0 = s.row_ptr[i], len = s.row_ptr[i + 1] - r0;
        for (int t = lane; t < C * K * n; t += 32) W[(long long)(t / n) * lsW + (long long)(t % n) * n + i] = 0.0;
        __syncwarp();
        for (int t = lane; t < C * K * len; t += 32) {
          const int ck = t / len, e = r0 + t % len;
          W[(long long)ck * lsW + (long long)s.col_idx[e] * n + i] = A[(long long)ck * lsA + e];
        }
        __syncwarp();
      }
    }
    __syncthreads();
    if (tr) tr[1] = gtimer();
    // ||b_k|| of the evaluated b (before the stage loop turns b into b')
    for (int k = warp; k < d; k += NT / 32) {
      R acc = md::zero<K>();
      for (int i = lane; i < n; i += 32) acc = md::add<K>(acc, S::absv(S::load(bb + (long long)k * n, lsV, i)));
      acc = md::group_sum<K>(acc, 32);
      if (lane == 0) md::store<K>(kn, d, k, acc);
    }
    // ---------------------------------------------------- Householder QR of [A_0 | I]
    {
      const int sub = tid % TPC;
      const int slots = (ncol + NT / TPC - 1) / (NT / TPC);  // column slots per lane group (uniform)
      // reflector c (column c, rows >= c) by one whole warp: alpha, v0, beta
      auto reflector = [&](int c) {
        Acc sg;
        S::acc_zero(sg);
        for (int r = c + lane; r < n; r += 32) S::acc_abs2(sg, S::load(W, lsW, (long long)c * n + r));
        S::acc_group(sg, 32);
        const R sig = S::rval(sg);
        const V x0 = S::load(W, lsW, (long long)c * n + c);
        const R nrm = md::sqrt<K>(sig);
        const R ax0 = S::absv(x0);
        const V alpha = S::neg(S::mul_real(S::phase(x0, ax0), nrm));
        const V v0 = S::sub(x0, alpha);
        R bt = md::zero<K>();
        if (!md::is_zero<K>(sig)) bt = md::recip<K>(md::mul<K>(nrm, md::add<K>(nrm, ax0)));
        __syncwarp();
        if (lane == 0) {
          S::store(vh, n, c, v0);
          md::store<K>(be, n, c, bt);
          S::store(W, lsW, (long long)c * n + c, alpha);
        }
      };
      if (warp == 0) reflector(0);
      __syncthreads();
      for (int j = 0; j < n; ++j) {
        const V v0 = S::load(vh, n, j);
        const R bt = md::load<K>(be, n, j);
        for (int sl = 0; sl < slots; ++sl) {
          // every lane takes part in the group shuffles (idle groups sum nothing)
          const int cg = sl * (NT / TPC) + tid / TPC;
          const bool act = cg < ncol && cg > j;
          Acc dt;
          S::acc_zero(dt);
          for (int r = j + sub; act && r < n; r += TPC) {
            const V v = (r == j) ? v0 : S::load(W, lsW, (long long)j * n + r);
            S::acc_prod(dt, S::conj(v), S::load(W, lsW, (long long)cg * n + r));
          }
          S::acc_group(dt, TPC);
          const V nw = S::neg(S::mul_real(S::val(dt), bt));
          for (int r = j + sub; act && r < n; r += TPC) {
            const V v = (r == j) ? v0 : S::load(W, lsW, (long long)j * n + r);
            const long long e = (long long)cg * n + r;
            S::store(W, lsW, e, S::fma(S::load(W, lsW, e), nw, v));
          }
        }
        // look-ahead: the warp holding column j+1 (updated by its own lane group
        // just now) forms reflector j+1 before the step's barrier: one barrier per
        // step instead of two
        if (j + 1 < n && warp == (((j + 1) % (NT / TPC)) * TPC) / 32) {
          __syncwarp();
          reflector(j + 1);
        }
        __syncthreads();
      }
    }
    if (tr) tr[2] = gtimer();
    // ---------------------------------------------------- inverses of R's diagonal tiles
    // inv([[A, B], [0, C]]) = [[inv A, -inv A B inv C], [0, inv C]] by doubling
    // sizes 2, 4, .., TB; R[r][c] = W[c][r]; scratch T1 in yv
    for (int t = 0; t < T; ++t) {
      const int t0 = t * TB, nb = min(TB, n - t0);
      double* Xt = RI + (long long)t * TT;
      for (int e = tid; e < TT; e += NT) {
        const int r = e / TB, c = e % TB;
        V v = S::zero();
        if (r == c) v = (r < nb) ? S::recip(S::load(W, lsW, (long long)(t0 + r) * n + t0 + r)) : S::one();
        S::store(Xt, lsI, e, v);
      }
      __syncthreads();
      for (int sz = 2; sz <= TB; sz <<= 1) {
        const int h = sz >> 1, nent = (TB / sz) * h * h;
        // T1[blk][p][q] = sum_{u=0}^{q} R[base+p][base+h+u] X[base+h+u][base+h+q]
        for (int e = tid; e < nent; e += NT) {
          const int blk = e / (h * h), pp = (e / h) % h, q = e % h, base = blk * sz;
          Acc a;
          S::acc_zero(a);
          for (int u = 0; u <= q; ++u) {
            const int rr = base + pp, cc = base + h + u;
            const V rv = (rr < nb && cc < nb) ? S::load(W, lsW, (long long)(t0 + cc) * n + t0 + rr) : S::zero();
            S::acc_prod(a, rv, S::load(Xt, lsI, (long long)cc * TB + base + h + q));
          }
          S::store(yv, lsY, e, S::val(a));
        }
        __syncthreads();
        // X[base+p][base+h+q] = - sum_{v=p}^{h-1} X[base+p][base+v] T1[blk][v][q]
        for (int e = tid; e < nent; e += NT) {
          const int blk = e / (h * h), pp = (e / h) % h, q = e % h, base = blk * sz;
          Acc a;
          S::acc_zero(a);
          for (int v = pp; v < h; ++v)
            S::acc_prod(a, S::load(Xt, lsI, (long long)(base + pp) * TB + base + v),
                        S::load(yv, lsY, (long long)blk * h * h + v * h + q));
          S::store(Xt, lsI, (long long)(base + pp) * TB + base + h + q, S::neg(S::val(a)));
        }
        __syncthreads();
      }
    }
    // one diagonal tile (n <= 32): M = R^-1 Q^H once, into the A_0 half of W (the
    // reflectors and R are no longer needed), so each stage is one matvec
    // dx_k = M b'_k (same algebra as y = Q^H b'_k, R dx_k = y) and two barriers
    const bool useM = (T == 1);
    if (useM) {
      for (int e = tid; e < n * n; e += NT) {
        const int r = e / n, j = e % n;
        Acc a;
        S::acc_zero(a);
        for (int c = r; c < n; ++c)
          S::acc_prod(a, S::load(RI, lsI, (long long)r * TB + c), S::load(W, lsW, (long long)(n + j) * n + c));
        S::store(W, lsW, (long long)j * n + r, S::val(a));
      }
      __syncthreads();
    }
    if (tr) tr[3] = gtimer();
    // ---------------------------------------------------- stage loop
    for (int k = 0; k < d; ++k) {
      if (useM) {  // dx_k = M b'_k, M[o][c] = W[c][o]
        for (int o0 = 0; o0 < n; o0 += NT / TPO) {
          const int o = o0 + tid / TPO, sub = tid % TPO;
          const bool act = o < n;
          Acc a;
          S::acc_zero(a);
          for (int c = sub; act && c < n; c += TPO)
            S::acc_prod(a, S::load(W, lsW, (long long)c * n + o), S::load(bb + (long long)k * n, lsV, c));
          S::acc_group(a, TPO);
          if (act && sub == 0) S::store(dxv + (long long)k * n, lsV, o, S::val(a));
        }
        __syncthreads();
      } else {
      // y = Q^H b'_k: (Q^H)[r][c] = W[n + c][r]
      for (int o0 = 0; o0 < n; o0 += NT / TPO) {  // uniform trip count: every lane joins the shuffles
        const int o = o0 + tid / TPO, sub = tid % TPO;
        const bool act = o < n;
        Acc a;
        S::acc_zero(a);
        for (int c = sub; act && c < n; c += TPO)
          S::acc_prod(a, S::load(W, lsW, (long long)(n + c) * n + o), S::load(bb + (long long)k * n, lsV, c));
        S::acc_group(a, TPO);
        if (act && sub == 0) S::store(yv, lsY, o, S::val(a));
      }
      __syncthreads();
      // R dx_k = y by tiles, last to first
      for (int t = T - 1; t >= 0; --t) {
        const int t0 = t * TB, t1 = min(n, t0 + TB);
        if (t < T - 1) {  // z = y - R[tile][> t1] dx_k[> t1]  (z kept in y)
          for (int o0 = t0; o0 < t1; o0 += NT / TPO) {
            const int o = o0 + tid / TPO, sub = tid % TPO;
            const bool act = o < t1;
            Acc a;
            S::acc_zero(a);
            for (int c = t1 + sub; act && c < n; c += TPO)
              S::acc_prod(a, S::load(W, lsW, (long long)c * n + o), S::load(dxv + (long long)k * n, lsV, c));
            S::acc_group(a, TPO);
            if (act && sub == 0) S::store(yv, lsY, o, S::sub(S::load(yv, lsY, o), S::val(a)));
          }
          __syncthreads();
        }
        for (int o0 = t0; o0 < t1; o0 += NT / TPO) {
          const int o = o0 + tid / TPO, sub = tid % TPO;
          const bool act = o < t1;
          Acc a;
          S::acc_zero(a);
          for (int c = t0 + sub; act && c < t1; c += TPO)
            S::acc_prod(a, S::load(RI + (long long)t * TT, lsI, (long long)(o - t0) * TB + (c - t0)),
                        S::load(yv, lsY, c));
          S::acc_group(a, TPO);
          if (act && sub == 0) S::store(dxv + (long long)k * n, lsV, o, S::val(a));
        }
        __syncthreads();
      }
      }
      // right-looking updates b'_{k'} -= A_{k'-k} dx_k, k' = k+1..D
      const int npairs = (d - 1 - k) * n;
      for (int pr = tid; pr < npairs; pr += NT) {
        const int kp = k + 1 + pr / n, i = pr % n;
        const int e0 = s.row_ptr[i], e1 = s.row_ptr[i + 1];
        Acc a;
        S::acc_zero(a);
        for (int e = e0; e < e1; ++e)
          S::acc_prod(a, S::load(A + (long long)(kp - k) * nnz, lsA, e),
                      S::load(dxv + (long long)k * n, lsV, s.col_idx[e]));
        const long long o = (long long)kp * n + i;
        S::store(bb, lsV, o, S::sub(S::load(bb, lsV, o), S::val(a)));
      }
      __syncthreads();
    }
    if (tr) tr[4] = gtimer();
    // ---------------------------------------------------- residual r_k = b'_k - A_0 dx_k (into bb), norms
    for (int pr = tid; pr < d * n; pr += NT) {
      const int k = pr / n, i = pr % n;
      Acc a;
      S::acc_zero(a);
      for (int e = s.row_ptr[i]; e < s.row_ptr[i + 1]; ++e)
        S::acc_prod(a, S::load(A, lsA, e), S::load(dxv + (long long)k * n, lsV, s.col_idx[e]));
      S::store(bb, lsV, pr, S::sub(S::load(bb, lsV, pr), S::val(a)));
    }
    __syncthreads();
    for (int kw = warp; kw < 2 * d; kw += NT / 32) {
      const int k = kw % d, w = 1 + kw / d;  // w = 1: r, 2: dx
      const double* src = (w == 1) ? bb : dxv;
      R acc = md::zero<K>();
      for (int i = lane; i < n; i += 32) acc = md::add<K>(acc, S::absv(S::load(src + (long long)k * n, lsV, i)));
      acc = md::group_sum<K>(acc, 32);
      if (lane == 0) md::store<K>(kn + (long long)w * K * d, d, k, acc);
    }
    // x += dx
    for (int t = tid; t < n * d; t += NT) {
      const int j = t / d, k = t % d;
      S::store(xg, lsX, t, S::add(S::load(xs, lsX, t), S::load(dxv + (long long)k * n, lsV, j)));
    }
    __syncthreads();
    if (RES && warp == 0 && lane < 3) {
      R best = md::zero<K>();
      for (int k = 0; k < d; ++k) {
        const R v = md::load<K>(kn + (long long)lane * K * d, d, k);
        if (md::greater<K>(v, best) || !isfinite(v.x[0])) best = v;
      }
      md::store<K>(RES + (size_t)p * K * 3, 3, lane, best);
    }
    __syncthreads();
    if (tr) tr[5] = gtimer();
  }
}

}  // namespace ns
