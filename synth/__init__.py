"""Seeded synthetic inputs for the Newton-step hot path (arxiv 2301.12659).

This module is shared by the oracle tests, the GPU parity tests and bench.py.
It holds NONE of the method's arithmetic: no series convolution, no
multiple-double (md) arithmetic, no evaluation/differentiation, no solve.
It only

* builds the paper's test systems as CSR monomial lists
  (one column of monomials x^E = b(t) with E lower-triangular ones,
  PAPER.md P:341-362 Eq.(5); the 2-column format c1 x^E1 + c2 x^E2 = b(t),
  P:416-448 Eq.(8)-(9), banded as DESIGN.md reading R9; the 1/(1-t) integer
  system, reading R13),
* writes the right-hand side r_i(t) from the CLOSED FORM of the exact
  solution: with x_j = exp(alpha_j t) (Eq.(6)) a monomial is
  exp(S t), S = sum of its alphas, whose coefficients are S^k/k!; with
  x_j = 1/(1-t) a monomial of m variables has coefficients C(k+m-1, m-1),
* draws the seeded perturbed starting series ('start', 'near'; reading R11),
* rounds exact rationals to md limbs limb by limb
  (limb_l = RN(v - sum_{<l} limbs)), using Python's correctly rounded
  int/int true division.

Layouts: x and rhs are limb-plane major
float64 arrays [K][n][d]; coefficients [K][M]; CSR arrays int32.
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass, field

import numpy as np

PREC_LIMBS = {"2d": 2, "4d": 4, "8d": 8}
LIMBS_NAME = {2: "2d", 4: "4d", 8: "8d"}
# T1 (tabMPneed) unit-roundoff constants: 2^-104, 2^-210, 2^-423
EPS_P = {2: 2.0 ** -104, 4: 2.0 ** -210, 8: 2.0 ** -423}
# north_star tolerances (BASELINE.json), relative to the running-error scale s_k
TOL_P = {2: 1e-28, 4: 1e-60, 8: 1e-120}
# half of the working precision for the 'start' input: ~sqrt(eps_p)
HALF_PREC = {2: 2.0 ** -52, 4: 2.0 ** -105, 8: 2.0 ** -211}


# --------------------------------------------------------------------------
# exact rational -> md limbs
# --------------------------------------------------------------------------
def rational_to_md(num: int, den: int, K: int) -> list[float]:
    """Round num/den (den > 0) to K nonoverlapping doubles, limb by limb.

    limb_0 = RN(v); limb_l = RN(v - limb_0 - ... - limb_{l-1}).  Python's
    int/int true division is correctly rounded, and the subtraction of a
    double from a rational is exact in integers.
    """
    out = []
    for _ in range(K):
        if num == 0:
            out.append(0.0)
            continue
        f = num / den
        if f == 0.0:  # below the double range: flush (reading R31)
            out.append(0.0)
            num = 0
            continue
        p, q = f.as_integer_ratio()  # q is a power of two
        num = num * q - p * den
        den = den * q
        out.append(f)
    return out


def frac_pair(x: float) -> tuple[int, int]:
    return x.as_integer_ratio()


# --------------------------------------------------------------------------
# systems
# --------------------------------------------------------------------------
@dataclass
class System:
    """A monomial system sum_{tau in eq i} c_tau x^tau = r_i(t) (Eq.(8)).

    Exponents are 0/1 (reading R8): a monomial is its strictly increasing
    variable list.  ``exact`` describes the closed-form solution used to
    write the rhs: ('exp', alphas) or ('inv1mt', None).
    """
    name: str
    n: int
    D: int
    K: int
    eq_ptr: np.ndarray      # int32 [n+1]
    mono_ptr: np.ndarray    # int32 [M+1]
    var_idx: np.ndarray     # int32 [sum m]
    coeff: np.ndarray       # float64 [K][M]  md coefficients (limb planes)
    rhs: np.ndarray         # float64 [K][n][d]
    exact: tuple
    meta: dict = field(default_factory=dict)
    is_complex: bool = False  # NEXT-2: coeff [2][K][M], rhs [2][K][n][d] (real planes, then imaginary)

    @property
    def d(self) -> int:
        return self.D + 1

    @property
    def M(self) -> int:
        return len(self.mono_ptr) - 1

    def monomials(self, i: int) -> list[int]:
        return list(range(int(self.eq_ptr[i]), int(self.eq_ptr[i + 1])))

    def variables(self, t: int) -> list[int]:
        return [int(v) for v in self.var_idx[self.mono_ptr[t]:self.mono_ptr[t + 1]]]

    def coeff_fraction_pairs(self, t: int) -> tuple[int, int]:
        # the exact value of the md coefficient: the sum of its limbs
        return _sum_pairs(frac_pair(float(v)) for v in self.coeff[:, t])


def _csr(eqs: list[list[list[int]]]):
    eq_ptr = [0]
    mono_ptr = [0]
    var_idx = []
    for monos in eqs:
        for vs in monos:
            assert list(vs) == sorted(vs) and len(vs) >= 1  # repeats = exponents > 1 (NEXT-3)
            var_idx.extend(vs)
            mono_ptr.append(len(var_idx))
        eq_ptr.append(len(mono_ptr) - 1)
    return (np.asarray(eq_ptr, np.int32), np.asarray(mono_ptr, np.int32),
            np.asarray(var_idx, np.int32))


def draw_alphas(n: int, seed: int, mode: str = "random") -> list[float]:
    """alpha in [-1,-1+delta] U [1-delta,1], delta = 1/8 (reading R10)."""
    if mode == "one":
        return [1.0] * n
    rng = np.random.Generator(np.random.PCG64(seed))
    mag = rng.uniform(7.0 / 8.0, 1.0, size=n)
    sgn = np.where(rng.integers(0, 2, size=n) == 0, -1.0, 1.0)
    return [float(s * m) for s, m in zip(sgn, mag)]


def _exp_coeff_rational(S_num: int, S_den: int, k: int) -> tuple[int, int]:
    """S^k / k! as an (unreduced) integer ratio."""
    return S_num ** k, (S_den ** k) * math.factorial(k)


def _sum_pairs(pairs):
    """exact sum of (num, den) pairs with power-of-two or factorial dens (unreduced)."""
    num, den = 0, 1
    for p, q in pairs:
        num = num * q + p * den
        den = den * q
    return num, den


def _alpha_sum(alphas, vs) -> tuple[int, int]:
    return _sum_pairs(frac_pair(alphas[v]) for v in vs)


def _rhs_exp_row(args):
    """row i of the exp rhs: [K][d] (a pure function of its inputs; a worker)."""
    Ss, cs, d, K = args
    out = np.zeros((K, d))
    for k in range(d):
        terms = []
        for (Sn, Sd), (cn, cd) in zip(Ss, cs):
            en, ed = _exp_coeff_rational(Sn, Sd, k)
            terms.append((cn * en, cd * ed))
        num, den = _sum_pairs(terms)
        out[:, k] = rational_to_md(num, den, K)
    return out


def _map_rows(fn, jobs):
    """map over equations; in parallel worker processes when the exact
    rational arithmetic is large (the configs C3/C4 take tens of seconds on
    one core).  Same values either way (each row is computed by fn alone)."""
    work = sum(len(j[0]) * j[2] * j[3] for j in jobs)  # (terms or coefficients) x d x K
    import multiprocessing as mp
    if work < 20000 or os.environ.get("SYNTH_SERIAL") or mp.current_process().daemon:
        return [fn(j) for j in jobs]
    ctx = mp.get_context("fork")
    procs = min(len(jobs), max(1, len(os.sched_getaffinity(0))))
    with ctx.Pool(procs) as pool:
        return pool.map(fn, jobs, chunksize=max(1, len(jobs) // (4 * procs)))


def _rhs_exp(eqs, coeffs, alphas, n, d, K) -> np.ndarray:
    """r_i,k = sum_tau c_tau S_tau^k / k!  (closed form of prod exp(alpha_j t))."""
    jobs = []
    t = 0
    for i, monos in enumerate(eqs):
        Ss = []
        cs = []
        for vs in monos:
            Ss.append(_alpha_sum(alphas, vs))
            cs.append(_cpair(coeffs[t]))
            t += 1
        jobs.append((Ss, cs, d, K))
    rows = _map_rows(_rhs_exp_row, jobs)
    rhs = np.zeros((K, n, d))
    for i, r in enumerate(rows):
        rhs[:, i, :] = r
    return rhs


def _rhs_inv1mt(eqs, coeffs, n, d, K) -> np.ndarray:
    """r_i,k = sum_tau c_tau C(k+m-1, m-1)  (prod of m copies of 1/(1-t))."""
    rhs = np.zeros((K, n, d))
    t = 0
    for i, monos in enumerate(eqs):
        for k in range(d):
            terms = []
            for j, vs in enumerate(monos):
                cn, cd = _cpair(coeffs[t + j])
                m = len(vs)
                terms.append((cn * math.comb(k + m - 1, m - 1), cd))
            num, den = _sum_pairs(terms)
            rhs[:, i, k] = rational_to_md(num, den, K)
        t += len(monos)
    return rhs


def _cpair(c) -> tuple[int, int]:
    """a coefficient given as a float (exact dyadic) or as an exact (num, den) pair"""
    return c if isinstance(c, tuple) else frac_pair(float(c))


def _coeff_planes(coeffs, K):
    """md coefficients [K][M], rounded limb by limb from their exact values."""
    c = np.zeros((K, len(coeffs)))
    for t, v in enumerate(coeffs):
        num, den = _cpair(v)
        c[:, t] = rational_to_md(num, den, K)
    return c


def triangular_system(n: int, D: int, K: int, seed: int = 0, alpha_mode: str = "random",
                      name: str = "TS1") -> System:
    """One column of monomials, E lower-triangular ones (Eq.(5)):
    equation i is x_0 x_1 ... x_i = r_i(t), exact solution x_j = exp(alpha_j t)."""
    eqs = [[list(range(i + 1))] for i in range(n)]
    coeffs = [1.0] * n
    alphas = draw_alphas(n, seed, alpha_mode)
    eq_ptr, mono_ptr, var_idx = _csr(eqs)
    rhs = _rhs_exp(eqs, coeffs, alphas, n, D + 1, K)
    return System(name, n, D, K, eq_ptr, mono_ptr, var_idx, _coeff_planes(coeffs, K), rhs,
                  ("exp", alphas), {"seed": seed, "alpha_mode": alpha_mode})


def banded_two_column_system(n: int, w: int, D: int, K: int, seed: int = 0,
                             name: str = "TS3") -> System:
    """2-column format c1 x^E1 + c2 x^E2 = b(t) (Eq.(8)-(9)), banded
    (reading R9): E1 row i = {max(0,i-w+1)..i}; E2 row i = E1 row n-1-i;
    c1 = 1, c2 = RN_md(v/3) with v ~ U[-3/2, 3/2] (so c2 ~ U[-1/2, 1/2]); the factor
    1/3 makes c2 a full md number (every limb nonzero; rounded limb by limb),
    so the coefficient limbs 1..K-1 are exercised; the rhs is that of the
    md-rounded c2, so exp(alpha_j t) is the exact solution (up to the rhs
    rounding)."""
    E1 = [list(range(max(0, i - w + 1), i + 1)) for i in range(n)]
    E2 = [E1[n - 1 - i] for i in range(n)]
    eqs = [[E1[i], E2[i]] if E1[i] != E2[i] else [E1[i]] for i in range(n)]
    rng = np.random.Generator(np.random.PCG64(seed + 7919))
    v = rng.uniform(-1.5, 1.5, size=n)
    coeffs = []
    for i in range(n):
        coeffs.append(1.0)
        if len(eqs[i]) == 2:
            vn, vd = frac_pair(float(v[i]))
            vn = vn - vn % 3 + 1  # numerator = 1 (mod 3): v/3 is not dyadic
            coeffs.append((vn, 3 * vd))
    # monomials must appear in ascending variable-list order inside the CSR?  No:
    # the order inside an equation is the summation order (reading R20).
    alphas = draw_alphas(n, seed)
    eq_ptr, mono_ptr, var_idx = _csr(eqs)
    planes = _coeff_planes(coeffs, K)
    # the rhs of the md-rounded coefficients (exp(alpha t) solves the system as stored)
    exact_c = [_sum_pairs(frac_pair(float(l)) for l in planes[:, t]) for t in range(len(coeffs))]
    rhs = _rhs_exp(eqs, exact_c, alphas, n, D + 1, K)
    return System(name, n, D, K, eq_ptr, mono_ptr, var_idx, planes, rhs,
                  ("exp", alphas), {"seed": seed, "w": w})


def inv1mt_system(n: int, D: int, K: int, two_column: bool = False,
                  name: str = "TS4") -> System:
    """Integer system: x_j = 1/(1-t) is the exact solution (reading R13).
    Every series coefficient of every product is an integer binomial, so
    eval/diff at integer inputs is bit-exact while values stay < 2^53."""
    E1 = [list(range(i + 1)) for i in range(n)]
    if two_column:
        E2 = [E1[n - 1 - i] for i in range(n)]
        eqs = [[E1[i], E2[i]] if E1[i] != E2[i] else [E1[i]] for i in range(n)]
        coeffs = []
        for i in range(n):
            coeffs.append(1.0)
            if len(eqs[i]) == 2:
                coeffs.append(2.0)
    else:
        eqs = [[E1[i]] for i in range(n)]
        coeffs = [1.0] * n
    eq_ptr, mono_ptr, var_idx = _csr(eqs)
    rhs = _rhs_inv1mt(eqs, coeffs, n, D + 1, K)
    return System(name, n, D, K, eq_ptr, mono_ptr, var_idx, _coeff_planes(coeffs, K), rhs,
                  ("inv1mt", None), {})


def custom_system(eqs: list[list[list[int]]], coeffs: list[float], D: int, K: int,
                  alphas: list[float], name: str = "custom") -> System:
    """Any monomial system with an exp(alpha t) exact solution; a variable
    listed e times in a monomial has exponent e (NEXT-3 general exponents)."""
    n = len(eqs)
    eq_ptr, mono_ptr, var_idx = _csr(eqs)
    rhs = _rhs_exp(eqs, coeffs, alphas, n, D + 1, K)
    return System(name, n, D, K, eq_ptr, mono_ptr, var_idx, _coeff_planes(coeffs, K), rhs,
                  ("exp", alphas), {})


# --------------------------------------------------------------------------
# starting series
# --------------------------------------------------------------------------
def exact_coeff_rational(system: System, j: int, k: int) -> tuple[int, int]:
    kind, alphas = system.exact
    if kind == "exp":
        an, ad = frac_pair(alphas[j])
        return _exp_coeff_rational(an, ad, k)
    if kind == "inv1mt":
        return 1, 1
    raise ValueError(kind)


def make_x(system: System, kind: str = "near", seed: int = 1) -> np.ndarray:
    """Starting series x, float64 [K][n][d] (reading R11).

    'exact': the closed-form solution rounded to md.
    'start': x_0 = exact_0 (1 + u h), higher coefficients 0, h = HALF_PREC[K]
             ("x_0 with half its precision correct").
    'near':  every coefficient x_k = exact_k (1 + u_k h).
    'rough': every coefficient x_k = exact_k (1 + u_k 2^-12): a step whose dx
             is far above the tolerance at every k, so parity on dx is never
             vacuous (tol_p s_k << |dx_k|).
    'int':   integer perturbation of the 1/(1-t) solution: x_{j,k} = 1 + (u in {0,1,2}).
    u ~ U[-1,1] from PCG64(seed).
    """
    n, d, K = system.n, system.d, system.K
    x = np.zeros((K, n, d))
    rng = np.random.Generator(np.random.PCG64(seed))
    h_num, h_den = frac_pair(HALF_PREC[K])
    if kind == "int":
        vals = rng.integers(0, 3, size=(n, d))
        x[0] = 1.0 + vals
        return x
    u = rng.uniform(-1.0, 1.0, size=(n, d))
    if kind == "rough":
        h_num, h_den = 1, 2 ** 12
    jobs = [([exact_coeff_rational(system, j, k) for k in range(d)], list(u[j]), d, K, kind, h_num, h_den)
            for j in range(n)]
    rows = _map_rows(_make_x_row, jobs)
    for j, r in enumerate(rows):
        x[:, j, :] = r
    return x


def _make_x_row(args):
    """series j of make_x: [K][d] (a worker; see make_x)."""
    exact, u, d, K, kind, h_num, h_den = args
    out = np.zeros((K, d))
    for k in range(d):
        if kind == "start" and k > 0:
            continue
        en, ed = exact[k]
        if kind == "exact":
            out[:, k] = rational_to_md(en, ed, K)
            continue
        un, ud = frac_pair(float(u[k]))
        # exact_k * (1 + u h) = en (ud h_den + un h_num) / (ed ud h_den)
        num = en * (ud * h_den + un * h_num)
        den = ed * ud * h_den
        out[:, k] = rational_to_md(num, den, K)
    return out


# --------------------------------------------------------------------------
# BASELINE.json configurations
# --------------------------------------------------------------------------
CONFIGS = {
    "C1": dict(kind="tri", n=8, D=8, K=2, seed=12661, alpha_mode="one",
               desc="dim=8 monomial test system, series degree 8, double-double, exp(t)"),
    "C2": dict(kind="tri", n=64, D=31, K=4, seed=12662, alpha_mode="random",
               desc="dim=64, degree 31, quad-double, one Newton step on one B200"),
    "C3": dict(kind="tri", n=128, D=63, K=8, seed=12663, alpha_mode="random",
               desc="dim=128, degree 63, octo-double"),
    "C4": dict(kind="band2", n=1024, w=32, D=31, K=4, seed=12664,
               desc="dim=1024 2-column banded (w=32) sparse-monomial system, degree 31, quad-double"),
    "C5": dict(kind="tri", n=32, D=15, K=2, seed=12665, batch=4096, alpha_mode="random",
               desc="batch of 4096 independent paths, dim=32, degree 15, double-double"),
}


def build_config(name: str, K: int | None = None, n: int | None = None, D: int | None = None,
                 seed_offset: int = 0) -> System:
    c = dict(CONFIGS[name])
    K = K or c["K"]
    n = n or c["n"]
    D = D if D is not None else c["D"]
    seed = c["seed"] + seed_offset
    if c["kind"] == "tri":
        return triangular_system(n, D, K, seed, c.get("alpha_mode", "random"), name=name)
    if c["kind"] == "band2":
        return banded_two_column_system(n, min(c["w"], n), D, K, seed, name=name)
    raise ValueError(name)


# --------------------------------------------------------------------------
# NEXT-2: complex coefficients
# --------------------------------------------------------------------------
def _cmul(a, b):
    return (a[0] * b[0] - a[1] * b[1], a[0] * b[1] + a[1] * b[0])


def unit_circle(count: int, seed: int) -> list[tuple[float, float]]:
    """count points (cos t, sin t), t ~ U[0, 2 pi) from PCG64(seed), rounded to
    doubles: "random complex numbers on the unit circle"; the
    rounded values are the exact inputs (|z| = 1 to within 2^-53)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    th = rng.uniform(0.0, 2.0 * math.pi, size=count)
    return [(float(math.cos(t)), float(math.sin(t))) for t in th]


def _cplanes(values, K, shape):
    """exact complex values (Fraction pairs) -> planes [2][K][...] rounded limb by limb"""
    out = np.zeros((2, K) + shape)
    flat = out.reshape(2, K, -1)
    for e, (re, im) in enumerate(values):
        flat[0, :, e] = rational_to_md(re.numerator, re.denominator, K)
        flat[1, :, e] = rational_to_md(im.numerator, im.denominator, K)
    return out


def complex_triangular_system(n: int, D: int, K: int, seed: int = 0, name: str = "TS1c") -> System:
    """The triangular system of Eq.(5) with complex data (NEXT-2):
    equation i is c_i x_0 x_1 ... x_i = r_i(t) with c_i and alpha_j on the unit
    circle; exact solution x_j = exp(alpha_j t), so r_i =
    c_i exp(S_i t), S_i = sum_{j<=i} alpha_j, coefficients c_i S_i^k / k! (exact
    Gaussian rationals, rounded limb by limb per component)."""
    from fractions import Fraction as Fr
    eqs = [[list(range(i + 1))] for i in range(n)]
    eq_ptr, mono_ptr, var_idx = _csr(eqs)
    alphas = unit_circle(n, seed)
    cs = unit_circle(n, seed + 104729)
    d = D + 1
    rhs_vals = []
    for i in range(n):
        S = (sum(Fr(alphas[j][0]) for j in range(i + 1)), sum(Fr(alphas[j][1]) for j in range(i + 1)))
        c = (Fr(cs[i][0]), Fr(cs[i][1]))
        p = c
        row = []
        for k in range(d):
            row.append((p[0] / math.factorial(k), p[1] / math.factorial(k)))
            p = _cmul(p, S)
        rhs_vals.append(row)
    rhs = _cplanes([v for row in rhs_vals for v in row], K, (n, d))
    coeff = _cplanes([(Fr(c[0]), Fr(c[1])) for c in cs], K, (n,))
    return System(name, n, D, K, eq_ptr, mono_ptr, var_idx, coeff, rhs, ("cexp", alphas), {"seed": seed},
                  is_complex=True)


def make_cx(system: System, kind: str = "near", seed: int = 1) -> np.ndarray:
    """Complex starting series [2][K][n][d] (reading R11 per component): 'exact'
    the rounded exp(alpha t); 'start' x_0 (1 + u h), higher coefficients 0;
    'near' / 'rough' every coefficient times (1 + u h), h = HALF_PREC[K] /
    2^-12, u ~ U[-1, 1] real from PCG64(seed)."""
    from fractions import Fraction as Fr
    n, d, K = system.n, system.d, system.K
    rng = np.random.Generator(np.random.PCG64(seed))
    u = rng.uniform(-1.0, 1.0, size=(n, d))
    h = Fr(1, 2 ** 12) if kind == "rough" else Fr(HALF_PREC[K])
    vals = []
    for j in range(n):
        a = (Fr(system.exact[1][j][0]), Fr(system.exact[1][j][1]))
        p = (Fr(1), Fr(0))
        for k in range(d):
            v = (p[0] / math.factorial(k), p[1] / math.factorial(k))
            if kind == "start" and k > 0:
                v = (Fr(0), Fr(0))
            elif kind != "exact":
                f = 1 + Fr(float(u[j, k])) * h
                v = (v[0] * f, v[1] * f)
            vals.append(v)
            p = _cmul(p, a)
    return _cplanes(vals, K, (n, d))
