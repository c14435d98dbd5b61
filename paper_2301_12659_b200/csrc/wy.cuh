// wy.cuh -- the solve half of the Newton step for large n (SURVEY 8(f) NEXT-3,
// P:113-126 blocked Householder / [Ver22], "8 blocks of size 128"
// at dimension 1024; blocks of 256 here, measured faster at C4): Q^T is never formed.
//
//   householder_qr_kernel (ncol = n)  R and the reflectors v_j, beta_j of A_0 only
//   wy_unpack_kernel      R and V row-major; the diagonal BW x BW blocks of R
//   wy_gram_kernel        S_p = striu(V_p^T V_p) + diag(1 / beta) per block of BW
//                         reflectors: the compact WY form H_j0 ... H_j0+BW-1 =
//                         I - V_p T_p V_p^T has T_p = S_p^{-1} (the forward
//                         recurrence T = [[T', -beta T' V'^T v], [0, beta]]
//                         inverts block-wise to [[T'^-1, V'^T v], [0, 1/beta]])
//   invert_upper_kernel   T_p = S_p^{-1} and the inverses of R's diagonal blocks
//                         (recursive doubling, as invert_tiles_kernel, in global memory)
//   stage_wy_kernel       per stage k: b'_k = b_k - sum_j A_j dx_{k-j}; then
//                         y = Q^T b'_k = (I - V_P T_P^T V_P^T) ... (I - V_0 T_0^T V_0^T) b'_k
//                         block by block (u = V_p^T y, u' = T_p^T u, y -= V_p u');
//                         R dx_k = y by BW-row tiles, last to first.
// Versus [A_0 | I] + M = R^{-1} Q^T: the QR does (2/3) n^3 instead of ~(5/3) n^3
// md multiply-adds and M (n^3 / 2) is not formed; a stage costs ~2.5 n^2 instead
// of n^2 md multiply-adds and 5 P + 1 grid barriers.
#pragma once
#include "common.cuh"
#include "solve.cuh"

namespace ns {

// sl += sum_t fa(t) fb(t) over t = t0, t0 + 32, ... < t1 (t0 includes the lane);
// the operands of WY_B consecutive terms are loaded before any is used (one L2
// round trip per batch instead of per term), alternating between two level
// accumulators (ILP), joined at the end in a fixed order.
__host__ __device__ constexpr int wy_batch(int K) { return K == 8 ? 1 : (K == 4 ? 2 : 4); }
template <int K, class FA, class FB>
__device__ __forceinline__ void lv_dot_strided(double (&sl)[K], int t0, int t1, FA fa, FB fb, int stride = 32) {
  constexpr int B = wy_batch(K);
  double s1[K];
  lv_zero<K>(s1);
  for (int t = t0; t < t1; t += stride * B) {
    md::mdv<K> a[B], b[B];
#pragma unroll
    for (int q = 0; q < B; ++q)
      if (t + stride * q < t1) {
        a[q] = fa(t + stride * q);
        b[q] = fb(t + stride * q);
      }
#pragma unroll
    for (int q = 0; q < B; ++q)
      if (t + stride * q < t1) {
        if (q & 1) lv_prod<K>(s1, a[q], b[q]);
        else lv_prod<K>(sl, a[q], b[q]);
      }
  }
#pragma unroll
  for (int q = 0; q < K; ++q) md::level_insert<K>(sl, q, s1[q]);
}

// R (row-major upper, diagonal alpha), V (row-major lower: V[r][j] = v_j[r],
// diagonal v0 = vhead) and the diagonal blocks of R (identity-padded) into
// blk[P + t] of the block array [K][2P][BW][BW].
template <int K>
__global__ void __launch_bounds__(256) wy_unpack_kernel(int n, int BW, int P, const double* __restrict__ W,
                                                        const double* __restrict__ vhead, double* R, double* V,
                                                        double* blk) {
  const long long nn = (long long)n * n;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x, nth = (long long)gridDim.x * blockDim.x;
  for (long long e = tid; e < nn; e += nth) {
    const int c = (int)(e / n), r = (int)(e % n);  // W order (coalesced reads), scattered writes
#pragma unroll
    for (int l = 0; l < K; ++l) {
      const double w = W[l * nn + e];
      R[l * nn + (long long)r * n + c] = (c >= r) ? w : 0.0;
      V[l * nn + (long long)r * n + c] = (r > c) ? w : ((r == c) ? vhead[(long long)l * n + c] : 0.0);
    }
  }
  const long long BB = (long long)BW * BW, lsB = 2LL * P * BB;
  for (long long e = tid; e < (long long)P * BB; e += nth) {
    const int t = (int)(e / BB), i = (int)((e % BB) / BW), c = (int)(e % BW);
    const int r = t * BW + i, cc = t * BW + c;
#pragma unroll
    for (int l = 0; l < K; ++l) {
      double v;
      if (r < n && cc < n) v = (c >= i) ? W[l * nn + (long long)cc * n + r] : 0.0;
      else v = (i == c && l == 0) ? 1.0 : 0.0;
      blk[l * lsB + (long long)P * BB + e] = v;
    }
  }
}

// S_p[i][l] (i <= l) = v_{j0+i}^T v_{j0+l} for i < l, 1 / beta_{j0+i} on the
// diagonal, identity beyond n; one warp per entry, lanes over the rows
// r >= j0 + l (v_l is zero above its row), unnormalised level sums.
// owner_beta: the beta slot holds beta; else alpha v0 = -1 / beta.
template <int K>
__global__ void __launch_bounds__(256) wy_gram_kernel(int n, int BW, int P, const double* __restrict__ W,
                                                      const double* __restrict__ vhead,
                                                      const double* __restrict__ beta, int owner_beta,
                                                      double* blk) {
  const long long nn = (long long)n * n, BB = (long long)BW * BW, lsB = 2LL * P * BB;
  const int lane = threadIdx.x & 31;
  const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long task = gw; task < (long long)P * BB; task += nw) {
    const int p = (int)(task / BB), i = (int)((task % BB) / BW), l = (int)(task % BW);
    const int j0 = p * BW, ji = j0 + i, jl = j0 + l;
    md::mdv<K> v;
    if (i > l) {
      v = md::zero<K>();
    } else if (jl >= n) {
      v = (i == l) ? md::from_double<K>(1.0) : md::zero<K>();
    } else if (i == l) {
      const md::mdv<K> bt = md::load<K>(beta, n, ji);
      if (owner_beta) v = md::is_zero<K>(bt) ? md::from_double<K>(1.0) : md::recip<K>(bt);
      else v = md::is_zero<K>(bt) ? md::from_double<K>(1.0) : md::neg<K>(bt);
    } else {
      double sl[K];
      lv_zero<K>(sl);
      lv_dot_strided<K>(
          sl, jl + lane, n, [&](int r) { return md::load<K>(W, nn, (long long)ji * n + r); },
          [&](int r) { return (r == jl) ? md::load<K>(vhead, n, jl) : md::load<K>(W, nn, (long long)jl * n + r); });
      v = md::group_sum_levels<K>(sl, 32);
    }
    if (lane == 0) md::store<K>(blk, lsB, task, v);
  }
}

// X_b = S_b^{-1} for the nblk upper-triangular BT x BT blocks of S ([K][nblk][BT][BT],
// row-major; limb stride nblk BT^2), by recursive doubling:
// inv([[A, B], [0, C]]) = [[inv A, -inv A B inv C], [0, inv C]], sizes 2, 4, ..., BT.
// One thread per output entry of each level (a serial dot of <= BT/2 terms as
// unnormalised level sums); T1: scratch of the same shape as X.
template <int K>
__global__ void __launch_bounds__(256) invert_upper_kernel(int nblk, int BT, const double* __restrict__ S, double* X,
                                                           double* T1, unsigned* bar) {
  GridBarrier gb(bar, 0u);
  const long long BB = (long long)BT * BT, ls = (long long)nblk * BB;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x, nth = (long long)gridDim.x * blockDim.x;
  for (long long e = tid; e < ls; e += nth) {
    const int i = (int)((e % BB) / BT), c = (int)(e % BT);
    md::store_cg<K>(X, ls, e, (i == c) ? md::recip<K>(md::load<K>(S, ls, e)) : md::zero<K>());
  }
  gb.sync();
  // each entry's dot (up to BT/2 terms) is shared by a group of IG lanes (lane s sums
  // the terms s, s + IG, ...; fixed butterfly): a serial dot per thread made the last
  // levels long chains (0.9 ms at C4)
  constexpr int IG = 8, OPW = 32 / IG;
  const int lane = threadIdx.x & 31, sub = lane % IG;
  const long long gw = tid >> 5, nw = nth >> 5;
  for (int sz = 2; sz <= BT; sz <<= 1) {
    const int h = sz >> 1;
    const long long per = (long long)(BT / sz) * h * h;
    for (long long base0 = gw * OPW; base0 < nblk * per; base0 += nw * OPW) {  // warp-uniform trip count
      const long long e = base0 + lane / IG;
      const bool ok = e < nblk * per;
      const long long b = ok ? e / per : 0, rr = ok ? e % per : 0;
      const int blk = (int)(rr / (h * h)), p = (int)((rr / h) % h), q = (int)(rr % h);
      const long long base = b * BB + (long long)blk * sz * (BT + 1);  // (blk sz, blk sz) of block b
      double sl[K];
      lv_zero<K>(sl);
      if (ok)
        for (int u = sub; u <= q; u += IG)
          lv_prod<K>(sl, md::load<K>(S, ls, base + (long long)p * BT + h + u),
                     md::load_cg<K>(X, ls, base + (long long)(h + u) * BT + h + q));
      const md::mdv<K> t = md::group_sum_levels<K>(sl, IG);
      if (ok && sub == 0) md::store_cg<K>(T1, ls, b * BB + rr, t);
    }
    gb.sync();
    for (long long base0 = gw * OPW; base0 < nblk * per; base0 += nw * OPW) {
      const long long e = base0 + lane / IG;
      const bool ok = e < nblk * per;
      const long long b = ok ? e / per : 0, rr = ok ? e % per : 0;
      const int blk = (int)(rr / (h * h)), p = (int)((rr / h) % h), q = (int)(rr % h);
      const long long base = b * BB + (long long)blk * sz * (BT + 1);
      double sl[K];
      lv_zero<K>(sl);
      if (ok)
        for (int v = p + sub; v < h; v += IG)
          lv_prod<K>(sl, md::load_cg<K>(X, ls, base + (long long)p * BT + v),
                     md::load_cg<K>(T1, ls, b * BB + (long long)blk * h * h + (long long)v * h + q));
      const md::mdv<K> t = md::group_sum_levels<K>(sl, IG);
      if (ok && sub == 0) md::store_cg<K>(X, ls, base + (long long)p * BT + h + q, md::neg<K>(t));
    }
    gb.sync();
  }
}

struct WyArgs {
  const double* b;    // [K][d][n]
  const double* A;    // [K][d][nnz]
  const double* W;    // [K][n][n] column-major: reflector j below its diagonal (column j)
  const double* V;    // [K][n][n] row-major V[r][j] = v_j[r]
  const double* vh;   // [K][n] v0 of each reflector
  const double* R;    // [K][n][n] row-major upper
  const double* X;    // [K][2P][BW][BW]: T_p (p < P), inverses of R's diagonal blocks (P + t)
  double* bp;         // [K][d][n]
  double* dx;         // [K][d][n]
  double* y;          // [K][n]
  double* part;       // [K][n][cmax] update chunk partials
  double* up;         // [K][BW] u = V_p^T y
  double* u;          // [K][BW] u' = T_p^T u
  int cmax, BW, P, k_lo;
};

template <int K>
__global__ void __launch_bounds__(256) stage_wy_kernel(DevSys s, WyArgs a, unsigned* bar) {
  __shared__ double red[K * 9];  // block_sum_levels scratch (8 warps + result)
  GridBarrier gb(bar, 0u);
  const int n = s.n, d = s.d, BW = a.BW, P = a.P;
  const int gw = gwarp(), nw = nwarps(), lane = lane_id();
  const long long lsV = (long long)d * n, nn = (long long)n * n, BB = (long long)BW * BW;
  const long long lsX = 2LL * P * BB;
  for (int k = a.k_lo; k < s.dc; ++k) {
    stage_updates<K>(s, a.b, a.A, a.dx, a.part, a.cmax, a.bp, a.y, k, a.k_lo, gb);
    gb.sync();
    double* dxk = a.dx + (long long)k * n;
    // ---- y = Q^T b'_k, block by block
    for (int p = 0; p < P; ++p) {
      const int j0 = p * BW, nbw = min(BW, n - j0);
      // u_l = v_{j0+l}^T y: one CTA per reflector, its threads split the rows (a
      // warp alone on a 1024-row dot waited ~240 cycles per term on its SMSP's
      // share of the FP64 pipe)
      for (int l = blockIdx.x; l < nbw; l += gridDim.x) {
        const int j = j0 + l;
        double s0[K];
        lv_zero<K>(s0);
        if (threadIdx.x == 0) lv_prod<K>(s0, md::load<K>(a.vh, n, j), md::load_cg<K>(a.y, n, j));
        lv_dot_strided<K>(
            s0, j + 1 + threadIdx.x, n, [&](int r) { return md::load<K>(a.W, nn, (long long)j * n + r); },
            [&](int r) { return md::load_cg<K>(a.y, n, r); }, blockDim.x);
        const md::mdv<K> t = block_sum_levels<K>(s0, red);
        if (threadIdx.x == 0) md::store_cg<K>(a.up, BW, l, t);
      }
      gb.sync();
      for (int i = gw; i < nbw; i += nw) {  // u'_i = sum_{l <= i} T[l][i] u_l
        double sl[K];
        lv_zero<K>(sl);
        lv_dot_strided<K>(
            sl, lane, i + 1, [&](int l) { return md::load<K>(a.X, lsX, (long long)p * BB + (long long)l * BW + i); },
            [&](int l) { return md::load_cg<K>(a.up, BW, l); });
        const md::mdv<K> t = md::group_sum_levels<K>(sl, 32);
        if (lane == 0) md::store_cg<K>(a.u, BW, i, t);
      }
      gb.sync();
      for (int r = j0 + gw; r < n; r += nw) {  // y_r -= sum_l V[r][j0+l] u'_l
        double sl[K];
        lv_zero<K>(sl);
        const int lmax = min(nbw, r - j0 + 1);
        lv_dot_strided<K>(
            sl, lane, lmax, [&](int l) { return md::load<K>(a.V, nn, (long long)r * n + j0 + l); },
            [&](int l) { return md::load_cg<K>(a.u, BW, l); });
        const md::mdv<K> t = md::group_sum_levels<K>(sl, 32);
        if (lane == 0) md::store_cg<K>(a.y, n, r, md::sub<K>(md::load_cg<K>(a.y, n, r), t));
      }
      gb.sync();
    }
    // ---- R dx_k = y, tiles of BW rows last to first
    for (int t = P - 1; t >= 0; --t) {
      const int t0 = t * BW, t1 = min(n, t0 + BW);
      if (t < P - 1) {  // z_r = y_r - sum_{c >= t1} R[r][c] dx_k[c]  (z kept in y)
        for (int r = t0 + blockIdx.x; r < t1; r += gridDim.x) {  // one CTA per row
          double sl[K];
          lv_zero<K>(sl);
          lv_dot_strided<K>(
              sl, t1 + threadIdx.x, n, [&](int c) { return md::load<K>(a.R, nn, (long long)r * n + c); },
              [&](int c) { return md::load_cg<K>(dxk, lsV, c); }, blockDim.x);
          const md::mdv<K> acc = block_sum_levels<K>(sl, red);
          if (threadIdx.x == 0) md::store_cg<K>(a.y, n, r, md::sub<K>(md::load_cg<K>(a.y, n, r), acc));
        }
        gb.sync();
      }
      for (int r = t0 + gw; r < t1; r += nw) {  // dx_k[r] = sum_{c in tile} inv(R_tt)[r][c] z_c
        double sl[K];
        lv_zero<K>(sl);
        lv_dot_strided<K>(
            sl, r + lane, t1,
            [&](int c) { return md::load<K>(a.X, lsX, (long long)(P + t) * BB + (long long)(r - t0) * BW + (c - t0)); },
            [&](int c) { return md::load_cg<K>(a.y, n, c); });
        const md::mdv<K> acc = md::group_sum_levels<K>(sl, 32);
        if (lane == 0) md::store_cg<K>(dxk, lsV, r, acc);
      }
      gb.sync();
    }
  }
}

}  // namespace ns

namespace ns {

// ---------------------------------------------------------------- Q^T from one WY block
// n <= 256 without the cluster QR (C3): the QR factors A_0 alone (n columns, not
// the 2n of [A_0 | I]: half the column updates on the reflector chain), then
// Q^T = I - V T^T V^T (one block, BW >= n) is formed by two parallel products and
// M = R^{-1} Q^T by form_m_kernel as before.  Lane groups of WY_G lanes per output
// entry (lane s sums the terms s, s + WY_G, ... as level sums, then a butterfly).
constexpr int WY_G = 8;

// Z = T^T V^T:  Z[l][c] = sum_{i <= min(l, c)} T[i][l] V[c][i]  (row-major n x n)
template <int K>
__global__ void __launch_bounds__(256) wy_z_kernel(int n, int BW, const double* __restrict__ X, long long lsX,
                                                   const double* __restrict__ V, double* Z) {
  const long long nn = (long long)n * n;
  const int lane = threadIdx.x & 31, sub = lane % WY_G;
  constexpr int OPW = 32 / WY_G;
  const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long base = gw * OPW; base < nn; base += nw * OPW) {
    const long long o = base + lane / WY_G;
    const bool ok = o < nn;
    const int l = ok ? (int)(o / n) : 0, c = ok ? (int)(o % n) : 0;
    double sl[K];
    lv_zero<K>(sl);
    if (ok)
      for (int i = sub; i <= min(l, c); i += WY_G)
        lv_prod<K>(sl, md::load<K>(X, lsX, (long long)i * BW + l), md::load<K>(V, nn, (long long)c * n + i));
    const md::mdv<K> z = md::group_sum_levels<K>(sl, WY_G);
    if (ok && sub == 0) md::store<K>(Z, nn, o, z);
  }
}

// Q^T = I - V Z:  Qt[r][c] = delta_rc - sum_{l <= r} V[r][l] Z[l][c]  (row-major n x n)
template <int K>
__global__ void __launch_bounds__(256) wy_qt_kernel(int n, const double* __restrict__ V, const double* __restrict__ Z,
                                                    double* Qt) {
  const long long nn = (long long)n * n;
  const int lane = threadIdx.x & 31, sub = lane % WY_G;
  constexpr int OPW = 32 / WY_G;
  const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long base = gw * OPW; base < nn; base += nw * OPW) {
    const long long o = base + lane / WY_G;
    const bool ok = o < nn;
    const int r = ok ? (int)(o / n) : 0, c = ok ? (int)(o % n) : 0;
    double sl[K];
    lv_zero<K>(sl);
    if (ok)
      for (int l = sub; l <= r; l += WY_G)
        lv_prod<K>(sl, md::load<K>(V, nn, (long long)r * n + l), md::load<K>(Z, nn, (long long)l * n + c));
    const md::mdv<K> t = md::group_sum_levels<K>(sl, WY_G);
    if (ok && sub == 0) md::store<K>(Qt, nn, o, md::sub<K>(md::from_double<K>(r == c ? 1.0 : 0.0), t));
  }
}

}  // namespace ns
