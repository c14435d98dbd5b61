"""Pins of the CPU oracle against what the paper and the mathematics fix.

-m "not gpu".  Each pin is chosen so that a plausible mistake in the oracle
(a dropped term, a wrong index, a transposed operand, a sign) fails one of
them.  None of these recompute the oracle's own formula.
"""
import math
import os
from fractions import Fraction

import numpy as np
import pytest
import sympy

import synth
from oracle import newton as O
from oracle import paper

GOLD = os.path.join(os.path.dirname(__file__), "golden")
FX = O.ExactField()


def _gold(name):
    rows = []
    with open(os.path.join(GOLD, name)) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                rows.append(line.split())
    return rows


# ---------------------------------------------------------------- paper values
def test_T1_inverse_factorials_as_printed():
    """T1: 1/k! printed to 2 digits; k=15 is the known garble (R27)."""
    for k, inv, _prec, _eps in _gold("T1_tabMPneed.txt"):
        k = int(k)
        true = 1.0 / math.factorial(k)
        printed = float(inv)
        if k == 15:
            assert abs(printed - true) / true < 0.015 and f"{true:.1e}" == "7.6e-13"
        else:
            assert f"{true:.1e}" == f"{printed:.1e}", (k, true, printed)


def test_T1_eps_are_powers_of_two():
    """T1 eps column = 2^-52, 2^-104, 2^-210, 2^-423, 2^-848."""
    want = {"2.2e-16": 52, "4.9e-32": 104, "6.1e-64": 210, "4.6e-128": 423, "5.3e-256": 848}
    for _k, _inv, _p, eps in _gold("T1_tabMPneed.txt"):
        if eps != "-":
            assert f"{2.0 ** -want[eps]:.1e}" == eps
    assert synth.EPS_P == {2: 2.0 ** -104, 4: 2.0 ** -210, 8: 2.0 ** -423}


def test_T1_precision_choice_vs_last_coefficient():
    """T1's rationale: the last coefficient 1/k! must exceed the working eps."""
    for k, _inv, prec, _eps in _gold("T1_tabMPneed.txt"):
        k = int(k)
        limbs = {"double": 1, "double_double": 2, "quad_double": 4, "octo_double": 8,
                 "hexa_double": 16}[prec]
        eps = {1: 2.0 ** -52, 2: 2.0 ** -104, 4: 2.0 ** -210, 8: 2.0 ** -423,
               16: 2.0 ** -848}[limbs]
        assert Fraction(1, math.factorial(k)) > Fraction(eps)


def test_T2_totals_and_eq16_factors():
    for limbs, a, s, m, tot in _gold("T2_tabcostmd.txt"):
        limbs, a, s, m, tot = map(int, (limbs, a, s, m, tot))
        assert a + s + m == tot == paper.T2[limbs][3]
    rows = _gold("eq16_factors.txt")
    for kind, key, val in rows:
        if kind == "factor":
            assert paper.T2[int(key)][3] / int(key) == float(val) == paper.INTENSITY_FACTORS[int(key)]
    assert round(84 / 11.5, 2) == 7.30 and round(217.75 / 84, 2) == 2.59


def test_eq12_job_list_and_count():
    """Eq.(12)/(13): m=4 gives exactly the printed 7 products."""
    fwd, bwd, cross = paper.reverse_mode_jobs(4)
    assert fwd == [("x1", "x2"), ("f1", "x3"), ("f2", "x4")]
    assert bwd == [("x4", "x3"), ("g1", "x2")]
    assert sorted(cross) == [(2, "x1", "g1"), (3, "f1", "x4")]
    assert len(_gold("eq12_m4_jobs.txt")) == 7
    for m in range(3, 40):
        f, b, c = paper.reverse_mode_jobs(m)
        assert len(f) + len(b) + len(c) == paper.products_per_monomial(m) == 3 * m - 5
    assert paper.products_per_monomial(1) == 0 and paper.products_per_monomial(2) == 1


def test_count_laws():
    """padded d^2 (S:201 d=5 -> 25) vs the triangular d(d+1)/2."""
    assert paper.padded_products(5) == 25
    for d in range(1, 70):
        a = [Fraction(1)] * d
        cnt = sum(k + 1 for k in range(d))
        assert paper.triangular_products(d) == cnt
    # SURVEY 8 closed form S(n) = 1.5n^2 - 3.5n + 2 for the one-column system
    for n in range(3, 50):
        S = sum(paper.products_per_monomial(m) for m in range(1, n + 1))
        assert 2 * S == 3 * n * n - 7 * n + 4


# ---------------------------------------------------------------- convolution
def test_conv_spec_examples():
    one_pt = [FX.one, FX.one, FX.zero]
    assert O.conv(one_pt, one_pt, 3, FX) == [1, 2, 1]
    e = [Fraction(1, math.factorial(k)) for k in range(4)]
    assert O.conv(e, e, 4, FX) == [1, 2, 2, Fraction(4, 3)]


def test_conv_exp_law_exact():
    """exp(at) exp(bt) = exp((a+b)t): coefficients (a+b)^k/k! exactly (binomial theorem)."""
    rng = np.random.default_rng(3)
    for _ in range(5):
        a, b = (Fraction(float(v)) for v in rng.uniform(-1, 1, 2))
        d = 12
        ea = [a ** k / math.factorial(k) for k in range(d)]
        eb = [b ** k / math.factorial(k) for k in range(d)]
        c = O.conv(ea, eb, d, FX)
        assert c == [(a + b) ** k / math.factorial(k) for k in range(d)]
        # operand order and a transposed index would break the law for a != b
        assert O.conv(eb, ea, d, FX) == c


def test_conv_binomial_law_exact():
    """(1-t)^-a (1-t)^-b = (1-t)^-(a+b): coefficients C(k+a+b-1, k)."""
    d = 15
    for a in range(1, 5):
        for b in range(1, 5):
            sa = [Fraction(math.comb(k + a - 1, k)) for k in range(d)]
            sb = [Fraction(math.comb(k + b - 1, k)) for k in range(d)]
            assert O.conv(sa, sb, d, FX) == [math.comb(k + a + b - 1, k) for k in range(d)]


# ---------------------------------------------------------------- eval / diff
def _exp_x(alphas, d):
    return [[Fraction(a) ** k / math.factorial(k) for k in range(d)] for a in alphas]


def test_monomial_value_and_partials_closed_form():
    """At x_j = exp(a_j t): value = exp(S t), d/dx_j = exp((S - a_j) t) (SURVEY c.5)."""
    rng = np.random.default_rng(5)
    alphas = [float(v) for v in rng.uniform(-1, 1, 6)]
    d = 8
    x = _exp_x(alphas, d)
    vs = [0, 2, 3, 5]
    S = sum(Fraction(alphas[v]) for v in vs)
    assert O.monomial_value(x, vs, d, FX) == [S ** k / math.factorial(k) for k in range(d)]
    for j in vs:
        Sj = S - Fraction(alphas[j])
        assert O.monomial_partial(x, vs, j, d, FX) == [Sj ** k / math.factorial(k) for k in range(d)]
    split = O.monomial_partials_split(x, vs, d, FX)
    assert split == [O.monomial_partial(x, vs, j, d, FX) for j in vs]


def test_partials_split_equals_definition_random():
    rng = np.random.default_rng(11)
    d = 6
    x = [[Fraction(float(v)) for v in rng.uniform(-2, 2, d)] for _ in range(7)]
    for vs in ([3], [1, 4], [0, 1, 2], [0, 2, 3, 5, 6], list(range(7))):
        assert O.monomial_partials_split(x, vs, d, FX) == \
            [O.monomial_partial(x, vs, j, d, FX) for j in vs]
    assert O.monomial_partial(x, [3], 3, d, FX) == O.unit_series(d, FX)  # m = 1 (R7)


def test_inv1mt_binomials_and_zero_residual():
    """x_j = 1/(1-t): monomial of m vars has coefficients C(k+m-1, m-1), partials
    C(k+m-2, m-2); b = 0 exactly at the exact solution (SURVEY c.5)."""
    sys_ = synth.inv1mt_system(8, 8, 2)
    x = synth.make_x(sys_, "exact")
    xs = O.read_x(x, FX)
    b, A = O.evaluate(sys_, xs, FX)
    for i in range(8):
        assert all(v == 0 for v in b[i])
        m = i + 1
        for j, ser in A[i].items():
            assert ser == [math.comb(k + m - 2, m - 2) if m >= 2 else (1 if k == 0 else 0)
                           for k in range(sys_.d)]
    assert max(math.comb(8 + 8 - 1, 7), 6435) == 6435  # C1 maximum (< 2^53)


def test_spec_A0_row_at_exact_solution():
    """n=3 lower-ones system at the exact solution: A0[2][j] = 1."""
    sys_ = synth.triangular_system(3, 3, 2, seed=1)
    xs = O.read_x(synth.make_x(sys_, "exact"), FX)
    b, A = O.evaluate(sys_, xs, FX)
    assert [A[2][j][0] for j in range(3)] == [1, 1, 1]


def test_two_column_equals_sum_of_columns():
    """Linearity: evaluating c1 x^E1 + c2 x^E2 = sum of the columns evaluated separately."""
    sys2 = synth.banded_two_column_system(6, 3, 4, 2, seed=3)
    xs = O.read_x(synth.make_x(sys2, "near", seed=4), FX)
    b, A = O.evaluate(sys2, xs, FX)
    rhs = O.read_rhs(sys2, FX)
    co = O.read_coeffs(sys2, FX)
    for i in range(6):
        tot = [FX.zero] * sys2.d
        for t in O.eq_monomials(sys2, i):
            v = O.monomial_value(xs, O.monomial_vars(sys2, t), sys2.d, FX)
            tot = [tot[k] + co[t] * v[k] for k in range(sys2.d)]
        assert b[i] == [rhs[i][k] - tot[k] for k in range(sys2.d)]


# ---------------------------------------------------------------- solve
def _dense_block(A, b, n, d):
    """Assemble Eq.(4) explicitly as an (nd) x (nd) sympy matrix."""
    M = sympy.zeros(n * d, n * d)
    rhs = sympy.zeros(n * d, 1)
    for k in range(d):
        for kk in range(k + 1):
            j = k - kk
            for i, row in A.items():
                for c, ser in row.items():
                    M[k * n + i, kk * n + c] = sympy.Rational(ser[j].numerator, ser[j].denominator)
        for i in range(n):
            rhs[k * n + i] = sympy.Rational(b[i][k].numerator, b[i][k].denominator)
    return M, rhs


def test_toeplitz_solve_vs_dense_block_system():
    """n=3, d=4 block forward substitution = dense 12x12 solve (sympy, exact)."""
    sys_ = synth.triangular_system(3, 3, 2, seed=7)
    xs = O.read_x(synth.make_x(sys_, "near", seed=8), FX)
    b, A = O.evaluate(sys_, xs, FX)
    dx = O.solve(A, b, 3, 4, FX)
    M, rhs = _dense_block(A, b, 3, 4)
    sol = M.LUsolve(rhs)
    for k in range(4):
        for i in range(3):
            assert Fraction(str(sol[k * 3 + i])) == dx[k][i]
    r = O.residual(A, b, dx, 3, 4, FX)
    assert all(v == 0 for rk in r for v in rk)


def test_toeplitz_solve_vs_numpy_two_column():
    sys_ = synth.banded_two_column_system(7, 3, 5, 2, seed=9)
    xs = O.read_x(synth.make_x(sys_, "near", seed=2), FX)
    b, A = O.evaluate(sys_, xs, FX)
    n, d = 7, 6
    dx = O.solve(A, b, n, d, FX)
    M, rhs = _dense_block(A, b, n, d)
    sol = np.linalg.solve(np.array(M.tolist(), dtype=float), np.array(rhs.tolist(), dtype=float))
    got = np.array([float(dx[k][i]) for k in range(d) for i in range(n)])
    assert np.allclose(got, sol[:, 0], rtol=1e-9, atol=1e-12)


def test_zero_rhs_gives_zero_update():
    """Eq.(11): QR dx_k = b_k = 0 => dx_k = 0."""
    sys_ = synth.triangular_system(4, 5, 2, seed=1)
    xs = O.read_x(synth.make_x(sys_, "near", seed=1), FX)
    _, A = O.evaluate(sys_, xs, FX)
    zero = {i: [FX.zero] * 6 for i in range(4)}
    dx = O.solve(A, zero, 4, 6, FX)
    assert all(v == 0 for dk in dx for v in dk)


def test_lower_ones_textbook_solve():
    """At x_j(0) = 1, A_0 of the triangular system is the lower-ones matrix L and
    (L^-1 b)_i = b_i - b_{i-1} (SURVEY c.5)."""
    sys_ = synth.triangular_system(6, 0, 2, seed=4)
    x = np.zeros((2, 6, 1)); x[0, :, 0] = 1.0
    xs = O.read_x(x, FX)
    b, A = O.evaluate(sys_, xs, FX)
    for i in range(6):
        for j in range(6):
            assert A[i].get(j, [0])[0] == (1 if j <= i else 0)
    dx = O.solve(A, b, 6, 1, FX)
    for i in range(6):
        assert dx[0][i] == b[i][0] - (b[i - 1][0] if i else 0)


# ---------------------------------------------------------------- Newton
def test_quadratic_convergence_and_fixed_point():
    """From 'start' (x_0 correct to half precision), iterated oracle
    steps converge to the closed form; coefficient k is exact to ~delta^(2^i - k)
    after i steps (SURVEY c.3).  At the exact solution the update is ~0."""
    F = O.MPField(600)
    n, D = 4, 7
    sys_ = synth.triangular_system(n, D, 8, seed=21)  # 8 limbs: rhs accurate to 2^-424
    exact = synth.make_x(sys_, "exact")
    ex = O.read_x(exact, F)
    x = synth.make_x(sys_, "start", seed=5).copy()
    # the oracle iterates on field values; keep x as field series
    xs = O.read_x(x, F)
    errs = []
    for it in range(1, 5):
        b, A = O.evaluate(sys_, xs, F)
        dx = O.solve(A, b, n, sys_.d, F)
        xs = [[xs[j][k] + dx[k][j] for k in range(sys_.d)] for j in range(n)]
        e = [max(abs(xs[j][k] - ex[j][k]) for j in range(n)) for k in range(sys_.d)]
        errs.append(e)
        good = 2 ** it - 2
        for k in range(min(good + 1, sys_.d)):
            assert e[k] < F.num(2.0 ** -380), (it, k, e[k])
    assert errs[-1][-1] < F.num(2.0 ** -380)
    # fixed point
    b, A = O.evaluate(sys_, ex, F)
    dx = O.solve(A, b, n, sys_.d, F)
    assert max(abs(v) for dk in dx for v in dk) < F.num(2.0 ** -400)


def test_step_norms_and_residual_exact():
    sys_ = synth.build_config("C1")
    x = synth.make_x(sys_, "near", seed=1)
    out = O.step(sys_, x, FX)
    assert out["norm_r"] == 0
    assert out["norm_b"] == max(sum(abs(out["b"][i][k]) for i in range(8)) for k in range(9))
    assert out["norm_dx"] > 0


def test_mp_tier_matches_exact_tier():
    sys_ = synth.triangular_system(5, 6, 4, seed=2)
    x = synth.make_x(sys_, "near", seed=3)
    ex = O.step(sys_, x, FX)
    F = O.field_for(4)
    hp = O.step(sys_, x, F)
    for k in range(7):
        for i in range(5):
            assert abs(F.to_fraction(hp["dx"][k][i]) - ex["dx"][k][i]) <= \
                Fraction(2) ** -480 * (1 + abs(ex["dx"][k][i]))


# ---------------------------------------------------------------- generator sanity
def test_rational_to_md_exact_and_nonoverlapping():
    rng = np.random.default_rng(0)
    for K in (2, 4, 8):
        for _ in range(50):
            num = int(rng.integers(1, 2 ** 62)) * 3 ** 40
            den = 7 ** 50
            limbs = synth.rational_to_md(num, den, K)
            rem = Fraction(num, den) - sum(Fraction(l) for l in limbs)
            assert abs(rem) <= abs(Fraction(limbs[-1])) * Fraction(2) ** -52
            for a, b in zip(limbs, limbs[1:]):
                assert b == 0 or abs(b) <= abs(a) * 2.0 ** -52


def test_exact_x_is_rounded_closed_form():
    sys_ = synth.triangular_system(3, 9, 4, seed=12)
    x = synth.make_x(sys_, "exact")
    a = Fraction(sys_.exact[1][1])
    for k in range(10):
        v = sum(Fraction(l) for l in x[:, 1, k])
        want = a ** k / math.factorial(k)
        assert abs(v - want) <= abs(want) * Fraction(2) ** -210


# ---------------------------------------------------------------- staggered (NEXT-1)
def test_staggered_orders_spec_examples():
    """Eq.(10) with floor division."""
    assert O.staggered_orders(64) == [1, 2, 4, 7, 11, 17, 26, 40, 61, 64]
    assert O.staggered_orders(4) == [1, 2, 4]
    assert O.staggered_orders(1) == [1]
    assert O.staggered_orders(32) == [1, 2, 4, 7, 11, 17, 26, 32]


def test_window_step_prefix_of_full_step():
    """Truncated products and the block lower-triangular solve: coefficients
    0..dc-1 of a step on the series truncated at t^dc equal those of the full
    step ("not all d coefficient vectors need to be involved");
    x_k, k >= dc, are untouched."""
    sys_ = synth.triangular_system(4, 6, 2, seed=3)
    x = synth.make_x(sys_, "near", seed=2)
    full = O.step(sys_, x, FX)
    for dc in (1, 3, 7):
        w = O.step_window(sys_, x, FX, 0, dc)
        for j in range(4):
            for k in range(sys_.d):
                want = full["x_new"][j][k] if k < dc else w["x"][j][k]
                assert w["x_new"][j][k] == want, (dc, j, k)


def test_window_retired_stages_exact_integer_system():
    """With x_0..x_{k_lo-1} exact, b_k = 0 there exactly, so the full step has
    dx_k = 0 for k < k_lo (Eq.(11)) and the windowed step [k_lo, d)
    equals it bit for bit; the retired coefficients stay frozen.  Integer
    system x_j = 1/(1-t) (exact rational arithmetic)."""
    sys_ = synth.inv1mt_system(4, 5, 2)
    x = synth.make_x(sys_, "exact").copy()
    x[0, :, 3:] += 0.25  # perturb coefficients >= 3 (dyadic, exact)
    full = O.step(sys_, x, FX)
    assert all(full["dx"][k][i] == 0 for k in range(3) for i in range(4))
    w = O.step_window(sys_, x, FX, 3, sys_.d)
    assert all(w["dx"][k][i] == 0 for k in range(3) for i in range(4))
    for j in range(4):
        for k in range(sys_.d):
            assert w["x_new"][j][k] == full["x_new"][j][k]
    assert w["norm_r"] == 0


def test_staggered_schedule_converges_to_closed_form():
    """Newton along the staggered schedule from 'start' reaches the
    closed form exp(alpha t) at every coefficient (quadratic convergence per
    order step, SURVEY c.3)."""
    F = O.MPField(600)
    n, D = 4, 7
    sys_ = synth.triangular_system(n, D, 8, seed=21)
    ex = O.read_x(synth.make_x(sys_, "exact"), F)
    x = synth.make_x(sys_, "start", seed=5)
    orders = O.staggered_orders(sys_.d) + [sys_.d] * 3
    for dc in orders:
        out = O.step_window(sys_, x, F, 0, dc)
        xs = out["x_new"]
        # back to limb planes: 8 limbs (2^-424) keep far more than the 2^-380 checked
        x = np.zeros_like(x)
        for j in range(n):
            for k in range(sys_.d):
                v = F.to_fraction(xs[j][k])
                num, den = v.numerator, v.denominator
                x[:, j, k] = synth.rational_to_md(num, den, 8)
    err = max(abs(F.from_limbs(x[:, j, k]) - ex[j][k]) for j in range(n) for k in range(sys_.d))
    assert err < F.num(2.0 ** -380), err


# ---------------------------------------------------------------- NEXT-4
def test_fabry_ratio_closed_forms():
    """Theorem 1: x = 1/(1 - t/rho) has c_k = rho^-k, so every
    ratio c_{k}/c_{k+1} is rho; exp(alpha t) has c_{D-1}/c_D = D/alpha exactly;
    a polynomial of degree < D has c_D = 0 (no finite singularity)."""
    for rho in (Fraction(3, 2), Fraction(-5, 7), Fraction(1, 2)):
        ser = [rho ** -k for k in range(10)]
        assert O.fabry_ratio(ser, FX) == rho
    alpha = Fraction(7, 8)
    D = 9
    ser = [alpha ** k / math.factorial(k) for k in range(D + 1)]
    assert O.fabry_ratio(ser, FX) == Fraction(D) / alpha
    assert O.fabry_ratio([Fraction(1), Fraction(2), Fraction(1), Fraction(0)], FX) is None


def test_fabry_ratio_tends_to_nearest_singularity():
    """Theorem 1's limit: for 1/((1 - t/rho)(1 - t/sigma)), |rho| < |sigma|,
    the ratio tends to the nearer singular point rho as the order grows."""
    rho, sigma = Fraction(1, 2), Fraction(3, 2)
    a = [rho ** -k for k in range(40)]
    b = [sigma ** -k for k in range(40)]
    errs = []
    for d in (8, 16, 32):
        ser = O.conv(a, b, d, FX)
        errs.append(abs(O.fabry_ratio(ser, FX) - rho))
    assert errs[0] > errs[1] > errs[2] and errs[2] < Fraction(1, 10 ** 5)


def test_sampled_residual_norm():
    """the residual of the selected equations; all equations give
    the full norm, a subset never exceeds it (sums of absolute values)."""
    r = [[Fraction(i - k, 3) for i in range(5)] for k in range(4)]
    assert O.residual_norm_sampled(r, range(5)) == O.series_norm(r)
    assert O.residual_norm_sampled(r, [1, 3]) == max(abs(Fraction(1 - k, 3)) + abs(Fraction(3 - k, 3)) for k in range(4))
    assert O.residual_norm_sampled(r, [2]) <= O.series_norm(r)


# ---------------------------------------------------------------- coefficients c != 1
def _exact_exp_x(sys_):
    """x_j = exp(alpha_j t) as exact rationals (not md-rounded): alpha_j^k / k!."""
    al = [Fraction(a) for a in sys_.exact[1]]
    return [[al[j] ** k / math.factorial(k) for k in range(sys_.d)] for j in range(sys_.n)]


def test_two_column_jacobian_closed_form_negative_coefficients():
    """2-column system c1 x^E1 + c2 x^E2 (Eq.(8)-(9)) with negative
    md coefficients c2: at x_j = exp(alpha_j t) a monomial tau is exp(S_tau t)
    and d/dx_j of it is exp((S_tau - alpha_j) t), so
        A_k[i][j] = sum_{tau in eq i, tau ∋ j} c_tau (S_tau - alpha_j)^k / k!
    (SURVEY c.5 closed form, summed with the signed coefficients), and
    b_i = r_i - sum_tau c_tau S_tau^k/k! is the rounding of the stored rhs only.
    A sign slip on c (abs(c), -c) or a dropped coefficient fails here."""
    sys_ = synth.banded_two_column_system(7, 3, 5, 4, seed=3)
    co = O.read_coeffs(sys_, FX)
    assert any(c < 0 for c in co) and any(c.denominator % 3 == 0 or c.denominator > 2 ** 60 for c in co)
    assert any(sys_.coeff[1:, t].any() for t in range(sys_.M))   # limbs 1..K-1 in use
    xs = _exact_exp_x(sys_)
    b, A = O.evaluate(sys_, xs, FX)
    al = [Fraction(a) for a in sys_.exact[1]]
    rhs = O.read_rhs(sys_, FX)
    for i in range(sys_.n):
        want = {}
        val = [Fraction(0)] * sys_.d
        for t in O.eq_monomials(sys_, i):
            vs = O.monomial_vars(sys_, t)
            S = sum(al[v] for v in vs)
            for k in range(sys_.d):
                val[k] += co[t] * S ** k / math.factorial(k)
            for j in vs:
                ser = want.setdefault(j, [Fraction(0)] * sys_.d)
                for k in range(sys_.d):
                    ser[k] += co[t] * (S - al[j]) ** k / math.factorial(k)
        assert A[i] == want, i
        for k in range(sys_.d):
            assert b[i][k] == rhs[i][k] - val[k]
            assert abs(b[i][k]) <= Fraction(2) ** -200 * (1 + abs(rhs[i][k]))


def test_newton_two_column_negative_coefficients_converges():
    """Quadratic convergence (SURVEY c.3) on the 2-column banded system with
    signed md coefficients c2: from 'start' the iterated oracle steps reach
    exp(alpha t) at coefficient k <= 2^i - 2 after i steps; a Jacobian with a
    wrong coefficient sign (e.g. abs(c)) gives a chord iteration that does not.
    From the exact solution the update is ~0 (fixed point)."""
    F = O.MPField(600)
    sys_ = synth.banded_two_column_system(6, 3, 6, 8, seed=11)
    assert any(float(sys_.coeff[0, t]) < 0 for t in range(sys_.M))
    n, d = sys_.n, sys_.d
    ex = O.read_x(synth.make_x(sys_, "exact"), F)
    xs = O.read_x(synth.make_x(sys_, "start", seed=5), F)
    for it in range(1, 5):
        b, A = O.evaluate(sys_, xs, F)
        dx = O.solve(A, b, n, d, F)
        xs = [[xs[j][k] + dx[k][j] for k in range(d)] for j in range(n)]
        for k in range(min(2 ** it - 1, d)):
            e = max(abs(xs[j][k] - ex[j][k]) for j in range(n))
            assert e < F.num(2.0 ** -380), (it, k, e)
    b, A = O.evaluate(sys_, ex, F)
    dx = O.solve(A, b, n, d, F)
    assert max(abs(v) for dk in dx for v in dk) < F.num(2.0 ** -400)


# ---------------------------------------------------------------- tolerance scales (SURVEY c.4)
def test_scales_hand_derived_inv1mt_and_negative_coefficient():
    """s_b and s_A at x_j = 1/(1-t) (every coefficient 1): a product of m
    variables has coefficients C(k+m-1, m-1), so for the triangular integer
    system (eq i = x_0..x_i, rhs the same product)
        s_b[k,i] = |r_i,k| + C(k+i, i) = 2 C(k+i, i),
        s_A[(i,j)][k] = C(k+i-1, i-1) (i >= 1),  s_A[(0,0)] = (1, 0, 0, ...).
    With a coefficient c = -1/2 on x_0 x_1 the scales carry |c| = 1/2."""
    sys_ = synth.inv1mt_system(4, 6, 2)
    x = synth.make_x(sys_, "exact")
    sc = O.scales(sys_, x)
    for i in range(4):
        for k in range(7):
            assert sc["s_b"][k, i] == 2 * math.comb(k + i, i)
            for j in range(i + 1):
                want = (1.0 if k == 0 else 0.0) if i == 0 else math.comb(k + i - 1, i - 1)
                assert sc["s_A"][(i, j)][k] == want, (i, j, k)
    sys2 = synth.custom_system([[[0]], [[0, 1]]], [1.0, -0.5], 5, 2, [1.0, 1.0])
    x2 = np.zeros((2, 2, 6)); x2[0] = 1.0
    sc2 = O.scales(sys2, x2)
    for k in range(6):
        assert sc2["s_b"][k, 1] == abs(sys2.rhs[0, 1, k]) + 0.5 * (k + 1)
        assert sc2["s_A"][(1, 0)][k] == 0.5 and sc2["s_A"][(1, 1)][k] == 0.5


def test_stage_scales_hand_derived_2x2():
    """The running-error recursion of SURVEY c.4 worked by hand on the
    integer system x_0 = r_0, x_0 x_1 = r_1 at x = 1/(1-t):
    A_0 = [[1,0],[1,1]], |A_0^-1| = [[1,0],[1,1]], s_A_j = [[0,0],[1,1]] (j >= 1),
    s_b_k = (2, 2(k+1)).  With dx = 0:  e = (2,4), (2,12), (2,28), s = 5, 13, 29.
    With dx_0 = (1, 0):                 e = (3,6), (2,16), (2,36), s = 7, 17, 37."""
    sys_ = synth.inv1mt_system(2, 2, 2)
    x = synth.make_x(sys_, "exact")
    sc = O.scales(sys_, x)
    A0 = np.array([[1.0, 0.0], [1.0, 1.0]])
    s, e = O.stage_scales(sys_, x, A0, np.zeros((3, 2)), sc["s_b"], sc["s_A"])
    assert list(s) == [5, 13, 29] and e.tolist() == [[2, 4], [2, 12], [2, 28]]
    dx = np.zeros((3, 2)); dx[0, 0] = 1.0
    s, e = O.stage_scales(sys_, x, A0, dx, sc["s_b"], sc["s_A"])
    assert list(s) == [7, 17, 37] and e.tolist() == [[3, 6], [2, 16], [2, 36]]


# ---------------------------------------------------------------- QR reuse (x0_factor)
def test_step_window_x0_factor():
    """step_window(x0_factor=...) factors the A_0 of an earlier x_0 (the QR
    "only once").  (1) With x0_factor = x it is the plain step, bit
    for bit.  (2) With another x_0 the stage-0 solve uses that matrix, worked
    by hand on x_0 = r_0, x_0 x_1 = r_1: A_0(x0f) = [[1,0],[x1f, x0f]], so
    dx_0 = (b_0, (b_1 - x1f b_0) / x0f); later stages use the same factor."""
    sys_ = synth.triangular_system(2, 3, 2, seed=4)
    x = synth.make_x(sys_, "near", seed=6)
    full = O.step_window(sys_, x, FX, 0, sys_.d)
    same = O.step_window(sys_, x, FX, 0, sys_.d, x0_factor=x)
    for key in ("dx", "x_new", "r"):
        assert full[key] == same[key], key
    xf = np.zeros((2, 2, 1)); xf[0, 0, 0] = 2.0; xf[0, 1, 0] = 3.0
    mod = O.step_window(sys_, x, FX, 0, sys_.d, x0_factor=xf)
    b = mod["b"]
    assert mod["dx"][0][0] == b[0][0]
    assert mod["dx"][0][1] == (b[1][0] - 3 * b[0][0]) / 2
    # stage 1: A_0(x0f) dx_1 = b_1 - A_1 dx_0 with the true A_1
    A1dx = O.matvec_sparse(mod["A"], 1, mod["dx"][0], 2, FX)
    r0, r1 = b[0][1] - A1dx[0], b[1][1] - A1dx[1]
    assert mod["dx"][1] == [r0, (r1 - 3 * r0) / 2]


# ---------------------------------------------------------------- NEXT-2: complex coefficients
def test_complex_generator_unit_circle_and_exact_rhs():
    """alpha_j and c_i on the unit circle (within 2^-52); the rhs is
    c_i S_i^k / k! exactly rounded per component (Gaussian rationals)."""
    sys_ = synth.complex_triangular_system(4, 5, 4, seed=3)
    for a in sys_.exact[1]:
        assert abs(a[0] ** 2 + a[1] ** 2 - 1.0) < 2.0 ** -50
    al = [complex(*a) for a in sys_.exact[1]]
    F = O.field_for(4, complex_=True)
    rhs = O.read_rhs(sys_, F)
    co = O.read_coeffs(sys_, F)
    for i in range(4):
        S = F.ctx.mpc(0)
        for j in range(i + 1):
            S += F.ctx.mpc(*sys_.exact[1][j])
        for k in range(6):
            want = co[i] * S ** k / F.ctx.factorial(k)
            assert abs(rhs[i][k] - want) <= F.ctx.mpf(2) ** -205 * (1 + abs(want))
    assert abs(abs(al[0]) - 1) < 1e-15


def test_complex_monomial_value_and_partials_closed_form():
    """At x_j = exp(alpha_j t), complex alpha on the unit circle: a monomial is
    exp(S t) and d/dx_j of it exp((S - alpha_j) t) (SURVEY c.5 closed form,
    the 4M products of P:630-648 computed by the oracle's truncated
    convolutions of complex series)."""
    F = O.ComplexMPField(800)
    al = synth.unit_circle(6, 9)
    d = 9
    x = [[F.ctx.mpc(*a) ** k / F.ctx.factorial(k) for k in range(d)] for a in al]
    vs = [0, 2, 3, 5]
    S = sum((F.ctx.mpc(*al[v]) for v in vs), F.ctx.mpc(0))
    tol = F.ctx.mpf(2) ** -700
    got = O.monomial_value(x, vs, d, F)
    for k in range(d):
        assert abs(got[k] - S ** k / F.ctx.factorial(k)) < tol
    for j in vs:
        Sj = S - F.ctx.mpc(*al[j])
        p = O.monomial_partial(x, vs, j, d, F)
        for k in range(d):
            assert abs(p[k] - Sj ** k / F.ctx.factorial(k)) < tol


def test_complex_solve_vs_numpy_dense_block_system():
    """Eq.(4) over C: the oracle's block forward substitution (complex LU with
    modulus pivoting) against numpy's complex dense solve of the (nd)x(nd)
    block system."""
    sys_ = synth.complex_triangular_system(4, 3, 2, seed=5)
    x = synth.make_cx(sys_, "rough", seed=6)
    F = O.field_for(2, complex_=True)
    b, A = O.evaluate(sys_, O.read_x(x, F), F)
    n, d = 4, 4
    dx = O.solve(A, b, n, d, F)
    M = np.zeros((n * d, n * d), complex)
    rhs = np.zeros(n * d, complex)
    for k in range(d):
        for kk in range(k + 1):
            for i, row in A.items():
                for c, ser in row.items():
                    M[k * n + i, kk * n + c] = complex(ser[k - kk])
        for i in range(n):
            rhs[k * n + i] = complex(b[i][k])
    sol = np.linalg.solve(M, rhs)
    got = np.array([complex(dx[k][i]) for k in range(d) for i in range(n)])
    assert np.allclose(got, sol, rtol=1e-9, atol=1e-12)
    r = O.residual(A, b, dx, n, d, F)
    assert max(abs(v) for rk in r for v in rk) < F.ctx.mpf(2) ** -200


def test_complex_newton_converges_and_fixed_point():
    """Quadratic convergence over C (SURVEY c.3) to exp(alpha t), alpha on the
    unit circle: coefficients k <= 2^i - 2 exact to the working precision after
    i steps; at the exact solution the update is ~0."""
    F = O.ComplexMPField(600)
    sys_ = synth.complex_triangular_system(4, 6, 8, seed=7)
    n, d = sys_.n, sys_.d
    ex = O.read_x(synth.make_cx(sys_, "exact"), F)
    xs = O.read_x(synth.make_cx(sys_, "start", seed=8), F)
    for it in range(1, 5):
        b, A = O.evaluate(sys_, xs, F)
        dx = O.solve(A, b, n, d, F)
        xs = [[xs[j][k] + dx[k][j] for k in range(d)] for j in range(n)]
        for k in range(min(2 ** it - 1, d)):
            assert max(abs(xs[j][k] - ex[j][k]) for j in range(n)) < F.ctx.mpf(2) ** -380, (it, k)
    b, A = O.evaluate(sys_, ex, F)
    dx = O.solve(A, b, n, d, F)
    assert max(abs(v) for dk in dx for v in dk) < F.ctx.mpf(2) ** -400


# ---------------------------------------------------------------- NEXT-3: general exponents (repeated variables)
def test_exponents_closed_forms():
    """x_j^e as e copies of j (reading R37): at x_j = exp(a_j t) the monomial
    is exp(S t), S = sum_j e_j a_j, and d/dx_j = e_j exp((S - a_j) t); at
    x_j = 1/(1-t) a monomial of total degree m has coefficients C(k+m-1, m-1)
    and d/dx_j = e_j C(k+m-2, m-2).  Both evaluate_row paths agree."""
    rng = np.random.default_rng(8)
    alphas = [float(v) for v in rng.uniform(-1, 1, 4)]
    d = 7
    x = _exp_x(alphas, d)
    vs = [0, 0, 0, 2, 3, 3]
    S = sum(Fraction(alphas[v]) for v in vs)
    assert O.monomial_value(x, vs, d, FX) == [S ** k / math.factorial(k) for k in range(d)]
    for j, e in ((0, 3), (2, 1), (3, 2)):
        Sj = S - Fraction(alphas[j])
        assert O.monomial_partial(x, vs, j, d, FX) == [e * Sj ** k / math.factorial(k) for k in range(d)]
    ones = [[Fraction(1)] * d for _ in range(4)]
    m = len(vs)
    assert O.monomial_value(ones, vs, d, FX) == [math.comb(k + m - 1, m - 1) for k in range(d)]
    assert O.monomial_partial(ones, vs, 3, d, FX) == [2 * math.comb(k + m - 2, m - 2) for k in range(d)]
    sys_ = synth.custom_system([[[0, 0, 1]], [[1, 1], [0]], [[0, 2, 2, 2]]], [1.0, -0.5, 1.0, 0.75], 5, 2,
                               [0.9, -0.95, 0.875])
    xs = O.read_x(synth.make_x(sys_, "rough", seed=3), FX)
    assert O.evaluate(sys_, xs, FX, split=True) == O.evaluate(sys_, xs, FX, split=False)


def test_exponents_newton_converges():
    """Quadratic convergence (SURVEY c.3) on a system with exponents up to 3."""
    F = O.MPField(600)
    sys_ = synth.custom_system([[[0, 0]], [[0, 1, 1]], [[1, 2, 2, 2]], [[0, 3], [2, 2]]],
                               [1.0, 1.0, -0.5, 0.75, 0.25], 6, 8, [0.9, -0.95, 0.875, -1.0])
    n, d = sys_.n, sys_.d
    ex = O.read_x(synth.make_x(sys_, "exact"), F)
    xs = O.read_x(synth.make_x(sys_, "start", seed=5), F)
    for it in range(1, 5):
        b, A = O.evaluate(sys_, xs, F)
        dx = O.solve(A, b, n, d, F)
        xs = [[xs[j][k] + dx[k][j] for k in range(d)] for j in range(n)]
        for k in range(min(2 ** it - 1, d)):
            assert max(abs(xs[j][k] - ex[j][k]) for j in range(n)) < F.num(2.0 ** -380), (it, k)
