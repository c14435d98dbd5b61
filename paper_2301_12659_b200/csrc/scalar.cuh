// scalar.cuh -- the scalar of a system: a real md number or a complex md
// number (NEXT-2), with the operations the batched Newton
// step needs, so one kernel source serves both.
//
// Memory: C = 1 (real) or 2 (complex) components of K limb planes each; value
// i of an array with limb-plane stride ls has component c, limb l at
// base[(c K + l) ls + i] (real planes first, then imaginary).
//
// Level accumulators (Acc): unnormalised level sums of md.cuh (prod_levels +
// level_insert, renormalised once by val()); a complex accumulator is two real
// ones.  The complex product is the 4M method of P:630-648:
//   (a + bi)(c + di) = (ac - bd) + (ad + bc) i,
// four real md products into the two accumulators (no Gauss/Karatsuba 3M:
// its cancellation breaks the componentwise error bound).
#pragma once
#include "md.cuh"

namespace ns {

template <int K>
MD_INL void lv_zero(double (&s)[K]) {
#pragma unroll
  for (int l = 0; l < K; ++l) s[l] = 0.0;
}
// s += a b (level sums, exact two_sum cascades, last level plain)
template <int K>
MD_INL void lv_prod(double (&s)[K], const md::mdv<K>& a, const md::mdv<K>& b) {
  double pl[K];
  md::prod_levels<K>(a, b, pl);
#pragma unroll
  for (int l = 0; l < K; ++l) md::level_insert<K>(s, l, pl[l]);
}
template <int K>
MD_INL void lv_add(double (&s)[K], const md::mdv<K>& a) {
#pragma unroll
  for (int l = 0; l < K; ++l) md::level_insert<K>(s, l, a.x[l]);
}
// butterfly over aligned groups of G lanes, symmetric operand order (lower lane
// first), so every lane of the group ends with the same bits
template <int K>
MD_INL void lv_group(double (&s)[K], int G) {
  const int lane = threadIdx.x & 31;
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
      for (int l = 0; l < K; ++l) md::level_insert<K>(s, l, hi_s[l]);
    }
  }
}

template <int K>
struct RealS {
  static constexpr int C = 1;
  using R = md::mdv<K>;  // real md (norms, beta)
  using V = md::mdv<K>;
  struct Acc {
    double s[K];
  };
  static MD_INL V zero() { return md::zero<K>(); }
  static MD_INL V one() { return md::from_double<K>(1.0); }
  static MD_INL V from_real(const R& r) { return r; }
  static MD_INL V load(const double* b, long long ls, long long i) { return md::load<K>(b, ls, i); }
  static MD_INL void store(double* b, long long ls, long long i, const V& v) { md::store<K>(b, ls, i, v); }
  static MD_INL V add(const V& a, const V& b) { return md::add<K>(a, b); }
  static MD_INL V sub(const V& a, const V& b) { return md::sub<K>(a, b); }
  static MD_INL V neg(const V& a) { return md::neg<K>(a); }
  static MD_INL V conj(const V& a) { return a; }
  static MD_INL V mul(const V& a, const V& b) { return md::mul<K>(a, b); }
  static MD_INL V mul_real(const V& a, const R& r) { return md::mul<K>(a, r); }
  static MD_INL V fma(const V& acc, const V& a, const V& b) { return md::fma_acc<K>(acc, a, b); }  // acc + a b
  static MD_INL V recip(const V& a) { return md::recip<K>(a); }
  static MD_INL R absv(const V& a) { return md::absv<K>(a); }
  static MD_INL bool is_zero(const V& a) { return md::is_zero<K>(a); }
  // x0 / |x0| with sign(0) = +1 (reading R13)
  static MD_INL V phase(const V& x0, const R&) { return md::from_double<K>(x0.x[0] < 0.0 ? -1.0 : 1.0); }
  static MD_INL bool nonfinite(const V& a) { return !isfinite(a.x[0]); }
  static MD_INL void acc_zero(Acc& a) { lv_zero<K>(a.s); }
  static MD_INL void acc_prod(Acc& a, const V& x, const V& y) { lv_prod<K>(a.s, x, y); }
  static MD_INL void acc_add(Acc& a, const V& v) { lv_add<K>(a.s, v); }
  static MD_INL void acc_group(Acc& a, int G) { lv_group<K>(a.s, G); }
  static MD_INL V val(const Acc& a) { return md::renorm<K, K>(a.s); }
  // |x|^2 into a real accumulator
  static MD_INL void acc_abs2(Acc& a, const V& x) { lv_prod<K>(a.s, x, x); }
  static MD_INL R rval(const Acc& a) { return md::renorm<K, K>(a.s); }
};

template <int K>
struct CplxS {
  static constexpr int C = 2;
  using R = md::mdv<K>;
  struct V {
    md::mdv<K> re, im;
  };
  struct Acc {
    double re[K], im[K];
  };
  static MD_INL V zero() { return V{md::zero<K>(), md::zero<K>()}; }
  static MD_INL V one() { return V{md::from_double<K>(1.0), md::zero<K>()}; }
  static MD_INL V from_real(const R& r) { return V{r, md::zero<K>()}; }
  static MD_INL V load(const double* b, long long ls, long long i) {
    return V{md::load<K>(b, ls, i), md::load<K>(b + (long long)K * ls, ls, i)};
  }
  static MD_INL void store(double* b, long long ls, long long i, const V& v) {
    md::store<K>(b, ls, i, v.re);
    md::store<K>(b + (long long)K * ls, ls, i, v.im);
  }
  static MD_INL V add(const V& a, const V& b) { return V{md::add<K>(a.re, b.re), md::add<K>(a.im, b.im)}; }
  static MD_INL V sub(const V& a, const V& b) { return V{md::sub<K>(a.re, b.re), md::sub<K>(a.im, b.im)}; }
  static MD_INL V neg(const V& a) { return V{md::neg<K>(a.re), md::neg<K>(a.im)}; }
  static MD_INL V conj(const V& a) { return V{a.re, md::neg<K>(a.im)}; }
  static MD_INL void acc_zero(Acc& a) {
    lv_zero<K>(a.re);
    lv_zero<K>(a.im);
  }
  // a += x y, the 4M product
  static MD_INL void acc_prod(Acc& a, const V& x, const V& y) {
    lv_prod<K>(a.re, x.re, y.re);
    lv_prod<K>(a.re, md::neg<K>(x.im), y.im);
    lv_prod<K>(a.im, x.re, y.im);
    lv_prod<K>(a.im, x.im, y.re);
  }
  static MD_INL void acc_add(Acc& a, const V& v) {
    lv_add<K>(a.re, v.re);
    lv_add<K>(a.im, v.im);
  }
  static MD_INL void acc_group(Acc& a, int G) {
    lv_group<K>(a.re, G);
    lv_group<K>(a.im, G);
  }
  static MD_INL V val(const Acc& a) { return V{md::renorm<K, K>(a.re), md::renorm<K, K>(a.im)}; }
  static MD_INL V mul(const V& a, const V& b) {
    Acc t;
    acc_zero(t);
    acc_prod(t, a, b);
    return val(t);
  }
  static MD_INL V mul_real(const V& a, const R& r) { return V{md::mul<K>(a.re, r), md::mul<K>(a.im, r)}; }
  static MD_INL V fma(const V& acc, const V& a, const V& b) {  // acc + a b
    Acc t;
    acc_zero(t);
    acc_prod(t, a, b);
    acc_add(t, acc);
    return val(t);
  }
  // |a|^2 = re^2 + im^2 into a real accumulator (its .re levels)
  static MD_INL void acc_abs2(Acc& a, const V& x) {
    lv_prod<K>(a.re, x.re, x.re);
    lv_prod<K>(a.re, x.im, x.im);
  }
  static MD_INL R rval(const Acc& a) { return md::renorm<K, K>(a.re); }
  static MD_INL R abs2(const V& a) {
    Acc t;
    acc_zero(t);
    acc_abs2(t, a);
    return rval(t);
  }
  static MD_INL R absv(const V& a) { return md::sqrt<K>(abs2(a)); }
  // 1/a = conj(a) / |a|^2
  static MD_INL V recip(const V& a) { return mul_real(conj(a), md::recip<K>(abs2(a))); }
  static MD_INL bool is_zero(const V& a) { return md::is_zero<K>(a.re) && md::is_zero<K>(a.im); }
  // x0 / |x0|, 1 for x0 = 0 (the complex Householder phase; R13 for real)
  static MD_INL V phase(const V& x0, const R& ax0) {
    if (md::is_zero<K>(ax0)) return one();
    return mul_real(x0, md::recip<K>(ax0));
  }
  static MD_INL bool nonfinite(const V& a) { return !isfinite(a.re.x[0]) || !isfinite(a.im.x[0]); }
};

}  // namespace ns
