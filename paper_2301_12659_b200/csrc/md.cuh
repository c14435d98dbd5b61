// md.cuh -- multiple-double (md) arithmetic on FP64 CUDA cores, sm_100a.
//
// A K-limb md number (K = 2 double-double, 4 quad-double, 8 octo-double) is an
// unevaluated sum of nonoverlapping doubles, most significant first
// (PAPER.md P:135-136).  Values live in registers as md<K>; in memory the
// limbs are stored as separate planes (structure of arrays, P:146-158,
// P:751-757) -- see layout.cuh.
//
// Every operation is built from the error-free transforms
//   two_sum   s + e = a + b exactly        (6 DADD)
//   two_prod  p + e = a * b exactly        (DMUL + DFMA)
// written with explicit round-to-nearest intrinsics so that the compiler can
// not contract or reassociate (reading R21).  There are no data
// dependent branches: renormalisation compacts zero limbs with predicated
// selects (integer pipe), the FP64 pipe sees a fixed instruction stream.
//
// Accuracy contract (normwise, the form the tolerance rule of SURVEY 8(c)
// c.4 needs): for the fused accumulate  r = acc + a*b
//   |r - (acc + a b)| <= c_K 2^(-53K) (|acc| + |a||b|),
// verified against exact rationals in tests/test_gpu_md.py.
//
// Costs (FP64 instructions, counted from this source):
//   K=2: fma_acc 14, mul 7, add 11
//   K=4: fma_acc ~140   K=8: fma_acc ~1000   (level cascade + renorm)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define MD_INL __device__ __forceinline__

namespace md {

// ---------------------------------------------------------------- EFTs
MD_INL double dadd(double a, double b) { return __dadd_rn(a, b); }
MD_INL double dsub(double a, double b) { return __dsub_rn(a, b); }
MD_INL double dmul(double a, double b) { return __dmul_rn(a, b); }
MD_INL double dfma(double a, double b, double c) { return __fma_rn(a, b, c); }

// Knuth two_sum: s = fl(a+b), e = a + b - s exactly.
MD_INL void two_sum(double a, double b, double& s, double& e) {
  s = dadd(a, b);
  double bb = dsub(s, a);
  e = dadd(dsub(a, dsub(s, bb)), dsub(b, bb));
}
// Dekker fast_two_sum, requires exponent(a) >= exponent(b) (or a == 0).
MD_INL void fast_two_sum(double a, double b, double& s, double& e) {
  s = dadd(a, b);
  e = dsub(b, dsub(s, a));
}
// two_prod with FMA: p = fl(a*b), e = a*b - p exactly.
MD_INL void two_prod(double a, double b, double& p, double& e) {
  p = dmul(a, b);
  e = dfma(a, b, -p);
}

template <int K>
struct mdv {
  double x[K];
};

template <int K>
MD_INL mdv<K> zero() {
  mdv<K> r;
#pragma unroll
  for (int i = 0; i < K; ++i) r.x[i] = 0.0;
  return r;
}
template <int K>
MD_INL mdv<K> from_double(double a) {
  mdv<K> r = zero<K>();
  r.x[0] = a;
  return r;
}
template <int K>
MD_INL mdv<K> neg(const mdv<K>& a) {
  mdv<K> r;
#pragma unroll
  for (int i = 0; i < K; ++i) r.x[i] = -a.x[i];
  return r;
}
template <int K>
MD_INL mdv<K> absv(const mdv<K>& a) {
  return a.x[0] < 0.0 ? neg(a) : a;
}

// ---------------------------------------------------------------- renormalisation
// Renormalize N doubles (roughly ordered by decreasing magnitude, possibly
// overlapping) into K nonoverlapping limbs.  Two passes, both with the exact
// two_sum (no ordering precondition):
//   1) VecSum bottom-up: s = x[N-1]; (s, e[i+1]) = two_sum(x[i], s); e[0] = s
//   2) top-down error distillation with zero compaction: carry eps = e[0];
//      (r, t) = two_sum(eps, e[i]); if t != 0 emit r and carry t, else carry r.
// This is the VecSum / VecSumErrBranch renormalisation of Joldes, Muller and
// Popescu (CAMPARY) with the branch replaced by predicated selects.
template <int K, int N>
MD_INL mdv<K> renorm(const double (&x)[N]) {
  double e[N];
  double s = x[N - 1];
#pragma unroll
  for (int i = N - 2; i >= 0; --i) two_sum(x[i], s, s, e[i + 1]);
  e[0] = s;
  mdv<K> out = zero<K>();
  double eps = e[0];
  int j = 0;  // number of limbs emitted
#pragma unroll
  for (int i = 1; i < N; ++i) {
    double r, t;
    two_sum(eps, e[i], r, t);
    const bool emit = (t != 0.0);
#pragma unroll
    for (int q = 0; q < K; ++q) {
      if (q < i) out.x[q] = (emit && j == q) ? r : out.x[q];
    }
    j += (emit && j < K) ? 1 : 0;
    eps = emit ? t : r;
  }
#pragma unroll
  for (int q = 0; q < K; ++q) out.x[q] = (j == q) ? eps : out.x[q];
  return out;
}

// ---------------------------------------------------------------- generic K
// Level accumulator: s[l] collects the terms of magnitude ~2^(-53 l) |scale|.
// insert(l, t) adds t exactly into s[l] with two_sum and cascades the rounding
// error down the levels; the last level s[K-1] is a plain sum (its rounding
// errors are of order 2^(-53 K) |scale| and are dropped, as are all terms of
// level >= K).
template <int K>
MD_INL void level_insert(double (&s)[K], int l, double t) {
#pragma unroll
  for (int q = 0; q < K - 1; ++q) {
    if (q >= l) two_sum(s[q], t, s[q], t);
  }
  s[K - 1] = dadd(s[K - 1], t);
}

// Level sums of the product a*b: the products a_i b_j with i + j = l and the
// two_prod errors of the products of level l - 1 enter level l; level K-1
// products are formed with FMA into the last level.  s is NOT normalised.
template <int K>
MD_INL void prod_levels(const mdv<K>& a, const mdv<K>& b, double (&s)[K]) {
  two_prod(a.x[0], b.x[0], s[0], s[1]);
#pragma unroll
  for (int l = 2; l < K; ++l) s[l] = 0.0;
#pragma unroll
  for (int l = 1; l < K - 1; ++l) {
#pragma unroll
    for (int i = 0; i <= l; ++i) {
      double p, e;
      two_prod(a.x[i], b.x[l - i], p, e);
      level_insert<K>(s, l, p);
      level_insert<K>(s, l + 1, e);
    }
  }
#pragma unroll
  for (int i = 0; i < K; ++i) s[K - 1] = dfma(a.x[i], b.x[K - 1 - i], s[K - 1]);
}

// Fused accumulate r = acc + a*b.  The product's level sums do not depend on
// acc; acc joins last (K level inserts + renorm), so in a dependent chain
// (a dot product) only the add is on the critical path and the next product
// overlaps it.  Cost K = 4: 20 two_sum + 6 two_prod + 4 FMA + 4 DADD + renorm;
// K = 8: 168 two_sum + 28 two_prod + 8 FMA + 8 DADD + renorm (csrc/md.cuh counts
// in perfmodel.py).
template <int K>
MD_INL mdv<K> fma_acc(const mdv<K>& acc, const mdv<K>& a, const mdv<K>& b) {
  double s[K];
  prod_levels<K>(a, b, s);
#pragma unroll
  for (int l = 0; l < K; ++l) level_insert<K>(s, l, acc.x[l]);
  return renorm<K, K>(s);
}

// Same operation with acc entering first (it seeds the level sums): shorter
// latency when the dependence runs through a or b (Newton iterations of
// recip / rsqrt), longer through acc.
template <int K>
MD_INL mdv<K> fma_acc_first(const mdv<K>& acc, const mdv<K>& a, const mdv<K>& b) {
  double s[K];
#pragma unroll
  for (int l = 0; l < K; ++l) s[l] = acc.x[l];
#pragma unroll
  for (int l = 0; l < K - 1; ++l) {
#pragma unroll
    for (int i = 0; i <= l; ++i) {
      double p, e;
      two_prod(a.x[i], b.x[l - i], p, e);
      level_insert<K>(s, l, p);
      level_insert<K>(s, l + 1, e);
    }
  }
#pragma unroll
  for (int i = 0; i < K; ++i) s[K - 1] = dfma(a.x[i], b.x[K - 1 - i], s[K - 1]);
  return renorm<K, K>(s);
}

// r = a + b with the same level accumulator.
template <int K>
MD_INL mdv<K> add(const mdv<K>& a, const mdv<K>& b) {
  double s[K];
#pragma unroll
  for (int l = 0; l < K; ++l) s[l] = a.x[l];
#pragma unroll
  for (int l = 0; l < K; ++l) level_insert<K>(s, l, b.x[l]);
  return renorm<K, K>(s);
}

template <int K>
MD_INL mdv<K> sub(const mdv<K>& a, const mdv<K>& b) {
  return add<K>(a, neg<K>(b));
}

template <int K>
MD_INL mdv<K> mul(const mdv<K>& a, const mdv<K>& b) {
  double s[K];
  prod_levels<K>(a, b, s);
  return renorm<K, K>(s);
}

// ---------------------------------------------------------------- double-double
// Specialisations for K = 2 (Dekker / Joldes-Muller-Popescu algorithms on FMA).
template <>
MD_INL mdv<2> fma_acc<2>(const mdv<2>& acc, const mdv<2>& a, const mdv<2>& b) {
  double p, e;
  two_prod(a.x[0], b.x[0], p, e);
  e = dfma(a.x[0], b.x[1], e);
  e = dfma(a.x[1], b.x[0], e);
  double s, t;
  two_sum(acc.x[0], p, s, t);
  t = dadd(t, dadd(acc.x[1], e));
  mdv<2> r;
  fast_two_sum(s, t, r.x[0], r.x[1]);
  return r;
}
template <>
MD_INL mdv<2> mul<2>(const mdv<2>& a, const mdv<2>& b) {
  double p, e;
  two_prod(a.x[0], b.x[0], p, e);
  e = dfma(a.x[0], b.x[1], e);
  e = dfma(a.x[1], b.x[0], e);
  mdv<2> r;
  fast_two_sum(p, e, r.x[0], r.x[1]);
  return r;
}
template <>
MD_INL mdv<2> add<2>(const mdv<2>& a, const mdv<2>& b) {
  double s, t;
  two_sum(a.x[0], b.x[0], s, t);
  t = dadd(t, dadd(a.x[1], b.x[1]));
  mdv<2> r;
  fast_two_sum(s, t, r.x[0], r.x[1]);
  return r;
}

// ---------------------------------------------------------------- division, sqrt
// Newton iterations with precision doubling (reading R23): the K-limb result
// refines the K/2-limb one, so the early iterations run in cheaper (shorter
// latency) arithmetic; each iteration is two or three fused accumulates.
template <int P, int K>
MD_INL mdv<P> trunc(const mdv<K>& a) {
  mdv<P> r;
#pragma unroll
  for (int i = 0; i < P; ++i) r.x[i] = (i < K) ? a.x[i] : 0.0;
  return r;
}

// 1/b: y = y_h + y_h (1 - b y_h), y_h = 1/b at K/2 limbs.  The residual
// e = 1 - b y_h is formed in K limbs; the correction y_h e only needs K/2 limbs
// (it is 2^(-53K/2) times smaller), so the critical path is
// recip<K/2> + fma<K> + mul<K/2> + add<K>.
template <int K>
MD_INL mdv<K> recip(const mdv<K>& b) {
  if constexpr (K == 2) {
    const double y0 = 1.0 / b.x[0];
    const mdv<2> e = fma_acc_first<2>(from_double<2>(1.0), neg<2>(b), from_double<2>(y0));
    mdv<2> r;
    fast_two_sum(y0, dmul(y0, e.x[0]), r.x[0], r.x[1]);
    return r;
  } else {
    const mdv<K / 2> yh = recip<K / 2>(trunc<K / 2, K>(b));
    const mdv<K> e = fma_acc_first<K>(from_double<K>(1.0), neg<K>(b), trunc<K, K / 2>(yh));
    const mdv<K / 2> corr = mul<K / 2>(yh, trunc<K / 2, K>(e));
    return add<K>(trunc<K, K / 2>(yh), trunc<K, K / 2>(corr));
  }
}

// sqrt(a), a >= 0: s = s_h + (a - s_h^2) / (2 s_h), s_h = sqrt at K/2 limbs; the
// residual in K limbs, the quotient in K/2 limbs (Karp-Markstein).  recip of
// 2 s_h runs alongside the residual.
template <int K>
MD_INL mdv<K> sqrt(const mdv<K>& a) {
  if (!(a.x[0] > 0.0)) return zero<K>();
  if constexpr (K == 2) {
    const double s0 = ::sqrt(a.x[0]);
    const mdv<2> r = fma_acc_first<2>(a, from_double<2>(-s0), from_double<2>(s0));
    mdv<2> out;
    fast_two_sum(s0, r.x[0] / (2.0 * s0), out.x[0], out.x[1]);
    return out;
  } else {
    const mdv<K / 2> sh = sqrt<K / 2>(trunc<K / 2, K>(a));
    mdv<K / 2> two_sh = sh;
#pragma unroll
    for (int i = 0; i < K / 2; ++i) two_sh.x[i] = 2.0 * sh.x[i];
    const mdv<K / 2> inv2 = recip<K / 2>(two_sh);
    const mdv<K> shK = trunc<K, K / 2>(sh);
    const mdv<K> r = fma_acc_first<K>(a, neg<K>(shK), shK);  // a - s_h^2
    const mdv<K / 2> corr = mul<K / 2>(trunc<K / 2, K>(r), inv2);
    return add<K>(shK, trunc<K, K / 2>(corr));
  }
}

// 1/sqrt(a) = recip(sqrt(a)) (not on a hot path)
template <int K>
MD_INL mdv<K> rsqrt(const mdv<K>& a) {
  return recip<K>(sqrt<K>(a));
}

// a / b = q + y (a - q b), q = a y, y = 1/b (Markstein correction)
template <int K>
MD_INL mdv<K> div(const mdv<K>& a, const mdv<K>& b) {
  const mdv<K> y = recip<K>(b);
  const mdv<K> q = mul<K>(a, y);
  const mdv<K> r = fma_acc_first<K>(a, neg<K>(q), b);
  return fma_acc_first<K>(q, y, r);
}

// sign of an md value (leading nonzero limb decides; limbs are nonoverlapping)
template <int K>
MD_INL bool is_negative(const mdv<K>& a) {
  return a.x[0] < 0.0;
}
template <int K>
MD_INL bool is_zero(const mdv<K>& a) {
  bool z = true;
#pragma unroll
  for (int i = 0; i < K; ++i) z = z && (a.x[i] == 0.0);
  return z;
}
// a > b ?
template <int K>
MD_INL bool greater(const mdv<K>& a, const mdv<K>& b) {
  mdv<K> d = sub<K>(a, b);
  return d.x[0] > 0.0;
}

// ---------------------------------------------------------------- multi-accumulator dot
// sum_{t in [t0, t1) step dt} x(t) * y(t) with NA independent accumulators
// (round robin, combined in a fixed order at the end): NA times the ILP of a
// single accumulation chain.  Deterministic for fixed (t0, t1, dt).
template <int K, int NA, typename F>
MD_INL mdv<K> dot_ilp(int t0, int t1, int dt, F term) {
  mdv<K> acc[NA];
#pragma unroll
  for (int a = 0; a < NA; ++a) acc[a] = zero<K>();
  int t = t0;
  for (; t + (NA - 1) * dt < t1; t += NA * dt) {
#pragma unroll
    for (int a = 0; a < NA; ++a) {
      mdv<K> x, y;
      term(t + a * dt, x, y);
      acc[a] = fma_acc<K>(acc[a], x, y);
    }
  }
#pragma unroll
  for (int a = 0; a < NA; ++a) {
    if (t + a * dt < t1) {
      mdv<K> x, y;
      term(t + a * dt, x, y);
      acc[a] = fma_acc<K>(acc[a], x, y);
    }
  }
#pragma unroll
  for (int a = 1; a < NA; ++a) acc[0] = add<K>(acc[0], acc[a]);
  return acc[0];
}

// ---------------------------------------------------------------- warp shuffles
template <int K>
MD_INL mdv<K> shfl_xor(const mdv<K>& a, int mask, int width = 32) {
  mdv<K> r;
#pragma unroll
  for (int i = 0; i < K; ++i) r.x[i] = __shfl_xor_sync(0xffffffffu, a.x[i], mask, width);
  return r;
}
template <int K>
MD_INL mdv<K> shfl(const mdv<K>& a, int src, int width = 32) {
  mdv<K> r;
#pragma unroll
  for (int i = 0; i < K; ++i) r.x[i] = __shfl_sync(0xffffffffu, a.x[i], src, width);
  return r;
}
// Butterfly sum over aligned groups of G lanes (G power of two <= 32).  Every
// lane of the group ends with the same bits (the tree is symmetric: lane and
// partner add in the same operand order, lower lane first).  For K >= 4 the
// intermediate sums stay as unnormalised level arrays (exact two_sum cascades,
// plain adds only in the last level) and are renormalised once at the end.
template <int K>
MD_INL mdv<K> group_sum(mdv<K> v, int G) {
  const int lane = threadIdx.x & 31;
  if constexpr (K == 2) {
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      if (off < G) {
        mdv<K> o = shfl_xor<K>(v, off);
        const bool hi = (lane & off) != 0;
        mdv<K> lo_v, hi_v;
#pragma unroll
        for (int i = 0; i < K; ++i) {
          lo_v.x[i] = hi ? o.x[i] : v.x[i];
          hi_v.x[i] = hi ? v.x[i] : o.x[i];
        }
        v = add<K>(lo_v, hi_v);
      }
    }
    return v;
  } else {
    double s[K];
#pragma unroll
    for (int i = 0; i < K; ++i) s[i] = v.x[i];
    bool any = false;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      if (off < G) {
        any = true;
        double o[K];
#pragma unroll
        for (int i = 0; i < K; ++i) o[i] = __shfl_xor_sync(0xffffffffu, s[i], off);
        const bool hi = (lane & off) != 0;
        double lo_s[K], hi_s[K];
#pragma unroll
        for (int i = 0; i < K; ++i) {
          lo_s[i] = hi ? o[i] : s[i];
          hi_s[i] = hi ? s[i] : o[i];
        }
#pragma unroll
        for (int i = 0; i < K; ++i) s[i] = lo_s[i];
#pragma unroll
        for (int l = 0; l < K; ++l) level_insert<K>(s, l, hi_s[l]);
      }
    }
    return any ? renorm<K, K>(s) : v;
  }
}

// group_sum of unnormalised level arrays (lane partial sums kept as levels):
// the same butterfly, one renormalisation at the end (also for G == 1).
template <int K>
MD_INL mdv<K> group_sum_levels(const double (&s0)[K], int G) {
  const int lane = threadIdx.x & 31;
  double s[K];
#pragma unroll
  for (int i = 0; i < K; ++i) s[i] = s0[i];
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    if (off < G) {
      double o[K];
#pragma unroll
      for (int i = 0; i < K; ++i) o[i] = __shfl_xor_sync(0xffffffffu, s[i], off);
      const bool hi = (lane & off) != 0;
      double lo_s[K], hi_s[K];
#pragma unroll
      for (int i = 0; i < K; ++i) {
        lo_s[i] = hi ? o[i] : s[i];
        hi_s[i] = hi ? s[i] : o[i];
      }
#pragma unroll
      for (int i = 0; i < K; ++i) s[i] = lo_s[i];
#pragma unroll
      for (int l = 0; l < K; ++l) level_insert<K>(s, l, hi_s[l]);
    }
  }
  return renorm<K, K>(s);
}

// ---------------------------------------------------------------- memory (limb planes)
// value i of a planar md array: limb l at base[l * stride + i]
template <int K>
MD_INL mdv<K> load(const double* base, long long stride, long long i) {
  mdv<K> r;
#pragma unroll
  for (int l = 0; l < K; ++l) r.x[l] = base[l * stride + i];
  return r;
}
// L2-coherent load (bypasses L1) for data written by other SMs in the same kernel
template <int K>
MD_INL mdv<K> load_cg(const double* base, long long stride, long long i) {
  mdv<K> r;
#pragma unroll
  for (int l = 0; l < K; ++l) r.x[l] = __ldcg(base + l * stride + i);
  return r;
}
template <int K>
MD_INL void store(double* base, long long stride, long long i, const mdv<K>& v) {
#pragma unroll
  for (int l = 0; l < K; ++l) base[l * stride + i] = v.x[l];
}
template <int K>
MD_INL void store_cg(double* base, long long stride, long long i, const mdv<K>& v) {
#pragma unroll
  for (int l = 0; l < K; ++l) __stcg(base + l * stride + i, v.x[l]);
}

}  // namespace md
