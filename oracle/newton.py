"""Plain, slow, obviously correct Newton step on truncated power series.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Imports nothing from the
product package.  Every function cites the passage of PAPER.md (P:line) it
follows.  Scalars are field elements supporting + - * / and abs(): exact
``fractions.Fraction`` (tier O-exact) or ``mpmath`` mpf in a private context
of ``prec`` bits (tier O-hp).  Series are Python lists of d scalars
(coefficient k = coefficient of t^k); the truncation drops t^{>=d}
(reading R5).
"""
from __future__ import annotations

from fractions import Fraction

import mpmath
import numpy as np


# --------------------------------------------------------------------------
# fields
# --------------------------------------------------------------------------
class ExactField:
    """Exact rationals.  md limbs are dyadic, so conversion is exact."""
    name = "exact"

    def __init__(self):
        self.zero = Fraction(0)
        self.one = Fraction(1)

    def num(self, f: float):
        return Fraction(f)

    def from_limbs(self, limbs):
        s = Fraction(0)
        for l in limbs:
            s += Fraction(float(l))
        return s

    def to_fraction(self, v):
        return v


class MPField:
    """mpmath at ``prec`` bits in a private context (no global state)."""

    def __init__(self, prec: int):
        self.ctx = mpmath.MPContext()
        self.ctx.prec = prec
        self.name = f"mp{prec}"
        self.zero = self.ctx.mpf(0)
        self.one = self.ctx.mpf(1)

    def num(self, f: float):
        return self.ctx.mpf(f)

    def from_limbs(self, limbs):
        # exact sum of dyadic limbs, rounded once to prec bits
        return self.num_fraction(sum((Fraction(float(l)) for l in limbs), Fraction(0)))

    def num_fraction(self, fr: Fraction):
        return self.ctx.mpf(fr.numerator) / self.ctx.mpf(fr.denominator)

    def to_fraction(self, v):
        sign, man, e, _bc = self.ctx.mpf(v)._mpf_   # value = (-1)^sign man 2^e
        m = -int(man) if sign else int(man)
        return Fraction(m * 2 ** e) if e >= 0 else Fraction(m, 2 ** (-e))


class ComplexMPField(MPField):
    """Complex scalars (NEXT-2): mpmath mpc at ``prec`` bits in a
    private context.  abs() is the modulus (pivoting, norms)."""
    is_complex = True

    def __init__(self, prec: int):
        super().__init__(prec)
        self.name = f"mpc{prec}"
        self.zero = self.ctx.mpc(0)
        self.one = self.ctx.mpc(1)

    def num(self, f):
        return self.ctx.mpc(f)

    def from_climbs(self, re_limbs, im_limbs):
        """exact sums of the dyadic limbs of each component, rounded once"""
        re = sum((Fraction(float(l)) for l in re_limbs), Fraction(0))
        im = sum((Fraction(float(l)) for l in im_limbs), Fraction(0))
        c = self.ctx
        return c.mpc(c.mpf(re.numerator) / c.mpf(re.denominator), c.mpf(im.numerator) / c.mpf(im.denominator))

    def to_fraction(self, v):
        """(re, im) as exact Fractions"""
        re = MPField.to_fraction(self, self.ctx.mpf(v.real))
        im = MPField.to_fraction(self, self.ctx.mpf(v.imag))
        return re, im


def field_for(K: int, exact: bool = False, complex_: bool = False):
    """O-exact, or O-hp at >= 2x the md bits (256 / 512 / 1024 for 2d / 4d / 8d);
    complex_: the complex O-hp field (NEXT-2)."""
    if complex_:
        return ComplexMPField({2: 256, 4: 512, 8: 1024}[K])
    if exact:
        return ExactField()
    return MPField({2: 256, 4: 512, 8: 1024}[K])


# --------------------------------------------------------------------------
# series (Eq.(14))
# --------------------------------------------------------------------------
def conv(a, b, d, F):
    """Truncated Cauchy product c_k = sum_{j=0}^{k} a_j b_{k-j}, k < d.

    Eq.(14) with the coefficients of negative index equal to
    zero; the paper's padded terms are zero products and are omitted
    (reading R6: same result)."""
    c = []
    for k in range(d):
        s = F.zero
        for j in range(k + 1):
            s = s + a[j] * b[k - j]
        c.append(s)
    return c


def unit_series(d, F):
    return [F.one] + [F.zero] * (d - 1)


def product(series_list, d, F):
    """prod of the series in list order, left to right; empty product = 1."""
    p = unit_series(d, F)
    for s in series_list:
        p = conv(p, s, d, F)
    return p


# --------------------------------------------------------------------------
# reading system inputs (synth.System duck type: n, D, d, K, eq_ptr, mono_ptr,
# var_idx, coeff [K][M], rhs [K][n][d])
# --------------------------------------------------------------------------
def read_x(x_planes, F):
    """x float64 [K][n][d] (limb planes), or [2][K][n][d] for a complex system
    (real planes, then imaginary) -> list of n series of field scalars."""
    if x_planes.ndim == 4:
        _, K, n, d = x_planes.shape
        return [[F.from_climbs(x_planes[0, :, j, k], x_planes[1, :, j, k]) for k in range(d)] for j in range(n)]
    K, n, d = x_planes.shape
    return [[F.from_limbs(x_planes[:, j, k]) for k in range(d)] for j in range(n)]


def read_coeffs(sys, F):
    if getattr(sys, "is_complex", False):
        return [F.from_climbs(sys.coeff[0, :, t], sys.coeff[1, :, t]) for t in range(sys.M)]
    return [F.from_limbs(sys.coeff[:, t]) for t in range(sys.M)]


def read_rhs(sys, F):
    return read_x(sys.rhs, F)


def monomial_vars(sys, t):
    return [int(v) for v in sys.var_idx[sys.mono_ptr[t]:sys.mono_ptr[t + 1]]]


def eq_monomials(sys, i):
    return range(int(sys.eq_ptr[i]), int(sys.eq_ptr[i + 1]))


def jacobian_pattern(sys):
    """Row i: sorted union of the variables of equation i's monomials (the
    structural nonzeros of A_k, k = 0..D; Eq.(8))."""
    rows = []
    for i in range(sys.n):
        s = set()
        for t in eq_monomials(sys, i):
            s.update(monomial_vars(sys, t))
        rows.append(sorted(s))
    return rows


# --------------------------------------------------------------------------
# evaluation and differentiation: the plain definition
# --------------------------------------------------------------------------
def monomial_value(x, vs, d, F):
    """prod_{j in tau} x_j(t), truncated."""
    return product([x[v] for v in vs], d, F)


def monomial_partial(x, vs, j, d, F):
    """d/dx_j prod_{l in tau} x_l.  With exponents 0/1 (reading R8) this is
    prod_{l in tau, l != j} x_l; the empty product is the series 1 (m = 1,
    reading R7).  A variable may repeat (x_j^e written as e copies of j: the
    general exponents of NEXT-3, reading R37): by the product rule
    the derivative is the sum over the occurrences of j of the product of all
    the other factors, i.e. e x_j^(e-1) prod_{l != j} x_l^(e_l)."""
    occ = [q for q, v in enumerate(vs) if v == j]
    tot = [F.zero] * d
    for q in occ:
        p = product([x[v] for r, v in enumerate(vs) if r != q], d, F)
        tot = [tot[k] + p[k] for k in range(d)]
    return tot


def monomial_partials_split(x, vs, d, F):
    """The partials of each occurrence (position q) of the monomial, written as
    the product of the factors before q times the product of the factors after q:
    prod_{l != j} x_l = (prod_{l < j} x_l) * (prod_{l > j} x_l).  The two
    factor lists are formed once (left to right, right to left).  Pinned
    against ``monomial_partial`` in tests/test_oracle.py; used only to keep
    the oracle affordable on large rows."""
    m = len(vs)
    before = [unit_series(d, F)]
    for q in range(m - 1):
        before.append(conv(before[-1], x[vs[q]], d, F))
    after = [unit_series(d, F)]
    for q in range(m - 1, 0, -1):
        after.append(conv(after[-1], x[vs[q]], d, F))
    after = after[::-1]  # after[q] = prod_{l > q} x_{v_l}
    return [conv(before[q], after[q], d, F) for q in range(m)]


def evaluate_row(sys, x, coeffs, rhs, i, d, F, split=False):
    """Row i of (b, A): b_i(t) = r_i(t) - sum_tau c_tau x^tau(t) (reading R3,
    P:317-319) and A[i][j](t) = sum_{tau ∋ j} c_tau d x^tau / d x_j, summed in
    ascending monomial order (reading R20).  Returns (b_i series,
    {j: series})."""
    val = [F.zero] * d
    row = {}
    for t in eq_monomials(sys, i):
        vs = monomial_vars(sys, t)
        c = coeffs[t]
        v = monomial_value(x, vs, d, F)
        val = [val[k] + c * v[k] for k in range(d)]
        if split:  # one partial per occurrence (positional), summed per variable below
            parts, owners = monomial_partials_split(x, vs, d, F), vs
        else:      # one partial per distinct variable (all its occurrences)
            owners = list(dict.fromkeys(vs))
            parts = [monomial_partial(x, vs, j, d, F) for j in owners]
        for j, p in zip(owners, parts):
            acc = row.get(j, [F.zero] * d)
            row[j] = [acc[k] + c * p[k] for k in range(d)]
    b = [rhs[i][k] - val[k] for k in range(d)]
    return b, row


def evaluate(sys, x, F, split=False, rows=None):
    """All rows (or the listed ``rows``): returns (b, A) with b[i] a series and
    A[i] a dict {j: series}.  x is a list of series (``read_x``)."""
    d = sys.d
    coeffs = read_coeffs(sys, F)
    rhs = read_rhs(sys, F)
    rows = range(sys.n) if rows is None else rows
    b, A = {}, {}
    for i in rows:
        b[i], A[i] = evaluate_row(sys, x, coeffs, rhs, i, d, F, split)
    return b, A


# --------------------------------------------------------------------------
# linear algebra
# --------------------------------------------------------------------------
def _abs(v):
    return abs(v)


def lu_factor(M, F):
    """Gaussian elimination with partial pivoting, textbook (Doolittle).
    Returns (LU, perm); raises ZeroDivisionError for a singular matrix."""
    n = len(M)
    a = [list(r) for r in M]
    perm = list(range(n))
    for c in range(n):
        p = max(range(c, n), key=lambda r: _abs(a[r][c]))
        if a[p][c] == 0:
            raise ZeroDivisionError(f"singular A0 at column {c}")
        if p != c:
            a[c], a[p] = a[p], a[c]
            perm[c], perm[p] = perm[p], perm[c]
        piv = a[c][c]
        for r in range(c + 1, n):
            l = a[r][c] / piv
            a[r][c] = l
            if l != 0:
                rc, rr = a[c], a[r]
                for q in range(c + 1, n):
                    rr[q] = rr[q] - l * rc[q]
    return a, perm


def lu_solve(LU, perm, rhs, F):
    n = len(LU)
    y = [rhs[perm[i]] for i in range(n)]
    for i in range(n):
        s = y[i]
        for q in range(i):
            s = s - LU[i][q] * y[q]
        y[i] = s
    for i in range(n - 1, -1, -1):
        s = y[i]
        for q in range(i + 1, n):
            s = s - LU[i][q] * y[q]
        y[i] = s / LU[i][i]
    return y


def dense_coeff(A, n, k, F):
    """Dense n x n matrix A_k from the row dicts (off-pattern zeros)."""
    M = [[F.zero] * n for _ in range(n)]
    for i, row in A.items():
        for j, s in row.items():
            M[i][j] = s[k]
    return M


def matvec_sparse(A, k, v, n, F):
    """(A_k v)_i over the structural entries of row i."""
    out = [F.zero] * n
    for i, row in A.items():
        s = F.zero
        for j, ser in row.items():
            s = s + ser[k] * v[j]
        out[i] = s
    return out


def solve(A, b, n, d, F, k_lo=0):
    """Block forward substitution of Eq.(4):
    for k = 0..d-1:  A_0 dx_k = b_k - sum_{j=1}^{k} A_j dx_{k-j}.
    Returns dx as a list of d coefficient vectors (each a list of n)."""
    LU, perm = lu_factor(dense_coeff(A, n, 0, F), F)
    dx = []
    for k in range(d):
        rhs = [b[i][k] for i in range(n)]
        for j in range(1, k + 1):
            Av = matvec_sparse(A, j, dx[k - j], n, F)
            rhs = [rhs[i] - Av[i] for i in range(n)]
        dx.append(lu_solve(LU, perm, rhs, F))
    return dx


def residual(A, b, dx, n, d, F):
    """r_k = b_k - sum_{j=0}^{k} A_j dx_{k-j}  ("report ||b(t) - A(t) dx(t)||")."""
    r = []
    for k in range(d):
        rk = [b[i][k] for i in range(n)]
        for j in range(0, k + 1):
            Av = matvec_sparse(A, j, dx[k - j], n, F)
            rk = [rk[i] - Av[i] for i in range(n)]
        r.append(rk)
    return r


def series_norm(vecs):
    """max over k of the vector 1-norm sum_i |v_k,i| (reading R16)."""
    return max(sum(abs(v) for v in vk) for vk in vecs)


def step(sys, x_planes, F, split=False):
    """One Newton step (P:316-323 body, one iteration, all orders 0..D):
    (A, b) := evaluate; dx := A \\ b; report ||b - A dx||; x := x + dx.
    Returns a dict of field-valued results."""
    n, d = sys.n, sys.d
    x = read_x(x_planes, F)
    b, A = evaluate(sys, x, F, split)
    dx = solve(A, b, n, d, F)
    r = residual(A, b, dx, n, d, F)
    x_new = [[x[i][k] + dx[k][i] for k in range(d)] for i in range(n)]
    bk = [[b[i][k] for i in range(n)] for k in range(d)]
    return dict(x=x, b=b, A=A, dx=dx, r=r, x_new=x_new,
                norm_b=series_norm(bk), norm_r=series_norm(r), norm_dx=series_norm(dx))


# --------------------------------------------------------------------------
# staggered computations
# --------------------------------------------------------------------------
def staggered_orders(d_max):
    """The order schedule of Eq.(10): d := d + 1 + d/2 with floor
    division (reading R19), from d = 1, capped at d_max."""
    out = [1]
    while out[-1] < d_max:
        out.append(min(d_max, out[-1] + 1 + out[-1] // 2))
    return out


def step_window(sys, x_planes, F, k_lo, dc, split=False, x0_factor=None):
    """One Newton step on the stage window [k_lo, dc): the system
    is evaluated and differentiated on the series truncated at t^dc (only the
    coefficients 0..dc-1 are "involved"); the retired stages
    k < k_lo take dx_k = 0 (Eq.(11): b_k = 0 => dx_k = 0); the
    active stages solve A_0 dx_k = b_k - sum_{j=1}^{k} A_j dx_{k-j}
    (Eq.(4)); x_k += dx_k for k < dc, x_k unchanged for k >= dc.  Norms are
    over k < dc.  ``x0_factor`` (limb planes [K][n][>=1]): factor the A_0 of
    that earlier x_0 instead (the QR "only once", reused while x_0 is frozen,
    P:665-668).  Returns the dict of ``step`` (dx and r have dc entries)."""
    n = sys.n
    x = read_x(x_planes, F)
    coeffs = read_coeffs(sys, F)
    rhs = read_rhs(sys, F)
    b, A = {}, {}
    for i in range(n):
        b[i], A[i] = evaluate_row(sys, x, coeffs, rhs, i, dc, F, split)
    A0src = A
    if x0_factor is not None:
        x0 = read_x(x0_factor[:, :, :1], F)
        A0src = {i: evaluate_row(sys, x0, coeffs, rhs, i, 1, F, split)[1] for i in range(n)}
    LU, perm = lu_factor(dense_coeff(A0src, n, 0, F), F)
    dx = []
    for k in range(dc):
        if k < k_lo:
            dx.append([F.zero] * n)
            continue
        rhs_k = [b[i][k] for i in range(n)]
        for j in range(1, k + 1):
            Av = matvec_sparse(A, j, dx[k - j], n, F)
            rhs_k = [rhs_k[i] - Av[i] for i in range(n)]
        dx.append(lu_solve(LU, perm, rhs_k, F))
    r = residual(A, b, dx, n, dc, F)
    x_new = [[x[i][k] + (dx[k][i] if k < dc else F.zero) for k in range(sys.d)] for i in range(n)]
    bk = [[b[i][k] for i in range(n)] for k in range(dc)]
    return dict(x=x, b=b, A=A, dx=dx, r=r, x_new=x_new,
                norm_b=series_norm(bk), norm_r=series_norm(r), norm_dx=series_norm(dx))


# --------------------------------------------------------------------------
# NEXT-4: residual sampling and the Fabry ratio
# --------------------------------------------------------------------------
def residual_norm_sampled(r, rows):
    """||r|| over the selected equations only: max over k of sum_{i in rows}
    |r_k,i| ("compute the residuals for those selected equations", P:918-921;
    norm of reading R16)."""
    return max(sum(abs(rk[i]) for i in rows) for rk in r)


def fabry_ratio(series, F):
    """c_{d-2} / c_{d-1} of a series with d coefficients: the ratio of
    Theorem 1 (Fabry) at the last two computed coefficients, an
    estimate of the nearest singular point z (radius |z|).  None
    when c_{d-1} = 0."""
    c_last = series[-1]
    if c_last == 0:
        return None
    return series[-2] / c_last


# --------------------------------------------------------------------------
# running-error scales -- float64 magnitudes only
# --------------------------------------------------------------------------
def _absconv(a, b, d):
    """truncated convolution of two magnitude series (float64)"""
    return np.convolve(a, b)[:d]


def _mag(planes):
    """float64 magnitudes of the leading limbs: |v| of [K][...] planes, the
    modulus of [2][K][...] complex planes"""
    return np.hypot(planes[0, 0], planes[1, 0]) if planes.ndim >= 2 and planes.shape[0] == 2 and \
        planes.ndim == 4 else np.abs(planes[0])


def scales(sys, x_planes):
    """Magnitude scales for the tolerance rule ||gpu - oracle|| <= tol_p * s
    (SURVEY.md 8(c) c.4), for the eval/diff outputs:

    s_b[k,i]      = |r_i,k| + sum_tau |c_tau| (conv_{j in tau} |x_j|)_k
    s_A[(i,j)][k] = sum_{tau ∋ j} |c_tau| (conv_{l in tau, l != j} |x_l|)_k

    float64 magnitudes of the leading limbs (they scale errors; they are not
    results)."""
    n, d = sys.n, sys.d
    cx = getattr(sys, "is_complex", False)
    xa = _mag(x_planes)                           # [n][d]
    ra = _mag(sys.rhs)
    ca = np.hypot(sys.coeff[0, 0], sys.coeff[1, 0]) if cx else np.abs(sys.coeff[0])
    s_b = np.zeros((d, n))
    s_A = {}
    one = np.zeros(d)
    one[0] = 1.0
    for i in range(n):
        acc = ra[i].copy()
        for t in eq_monomials(sys, i):
            vs = monomial_vars(sys, t)
            m = len(vs)
            # |.|-products before and after each occurrence q: the partial of
            # occurrence q is pre[q] * suf[q + 1] (summed per variable, as the
            # partials themselves; repeated variables = exponents, R37)
            pre = [one]
            for v in vs:
                pre.append(_absconv(pre[-1], xa[v], d))
            suf = [one] * (m + 1)
            for q in range(m - 1, -1, -1):
                suf[q] = _absconv(suf[q + 1], xa[vs[q]], d)
            acc += ca[t] * pre[m]
            for q, j in enumerate(vs):
                s_A[(i, j)] = s_A.get((i, j), np.zeros(d)) + ca[t] * _absconv(pre[q], suf[q + 1], d)
        s_b[:, i] = acc
    return dict(s_b=s_b, s_A=s_A)


def stage_scales(sys, x_planes, A0_float, dx_float, s_b, s_A):
    """Running-error scale of the stage solve:
      m_k = s_b_k + sum_{j=1}^{k} (s_A_j |dx_{k-j}| + |A_j| e_{k-j}) + s_A_0 |dx_k|
      e_k = |A_0^{-1}| m_k ;   s_k = max_i (e_k,i + |x_k,i| + |dx_k,i|)
    |A_j| is bounded by s_A_j (the same sums of absolute products).  Inputs are
    float64: A_0 [n][n] (for |A_0^{-1}|), dx [d][n]."""
    n, d = sys.n, sys.d
    SA = np.zeros((d, n, n))
    for (i, j), ser in s_A.items():
        SA[:, i, j] = ser
    inv_abs = np.abs(np.linalg.inv(A0_float))
    dxa = np.abs(dx_float)
    xa = _mag(x_planes).T                          # [d][n]
    e = np.zeros((d, n))
    s = np.zeros(d)
    for k in range(d):
        m = s_b[k].copy()
        for j in range(1, k + 1):
            m += SA[j] @ dxa[k - j] + SA[j] @ e[k - j]
        m += SA[0] @ dxa[k]
        e[k] = inv_abs @ m
        s[k] = np.max(e[k] + xa[k] + dxa[k])
    return s, e
