"""Row a0: the device md arithmetic against exact rationals (T0 of SURVEY 4.2).

Every result is compared with the exact Fraction value of the operation on the
exact (dyadic) inputs; the bound is normwise, the form the tolerance rule
needs: |r - exact| <= C eps_p (|a| + |b|) for add, eps_p |a b| for mul,
eps_p (|c| + |a b|) for the fused accumulate (eps_p from T1: 2^-104, 2^-210,
2^-423).  Also: outputs are nonoverlapping, runs are deterministic.
"""
import math
from fractions import Fraction

import numpy as np
import pytest

import synth
from tests.helpers import gpu_available, limbs_to_fraction

pytestmark = pytest.mark.gpu

N_RANDOM = 4000


def _md_from_rational(num, den, K):
    return synth.rational_to_md(num, den, K)


def _inputs(K, n, seed, kind):
    """random md numbers: a random rational of ~60+ bits of structure (so all K
    limbs are used) scaled by 2^e, e in [-60, 60] ('rand') or [-250, 250]
    ('wide'; products stay inside the double range); 'int' mixes in
    integers (short expansions with zero limbs)."""
    rng = np.random.default_rng(seed)
    out = np.zeros((K, n))
    span = 60 if kind != "wide" else 250
    for i in range(n):
        den = 7 ** int(rng.integers(40, 200)) * 5 ** int(rng.integers(0, 30))
        num = den + int.from_bytes(rng.bytes(80), "little") % den    # value in [1, 2)
        e = int(rng.integers(-span, span))
        if e >= 0:
            num <<= e
        else:
            den <<= -e
        if rng.integers(0, 2):
            num = -num
        if kind == "int" and i % 2 == 0:
            num, den = int(rng.integers(-2 ** 40, 2 ** 40)), 1
        out[:, i] = _md_from_rational(num, den, K)
    return out


def _run(K, op, a, b=None, c=None):
    import torch
    import paper_2301_12659_b200 as P
    ta = torch.tensor(a, device="cuda:0")
    tb = None if b is None else torch.tensor(b, device="cuda:0")
    tc = None if c is None else torch.tensor(c, device="cuda:0")
    r = P.md_op(K, op, ta, tb, tc)
    torch.cuda.synchronize()
    return r.cpu().numpy()


def _check_nonoverlap(r):
    K, n = r.shape
    for i in range(n):
        for l in range(K - 1):
            hi, lo = r[l, i], r[l + 1, i]
            if lo != 0:
                assert hi != 0 and abs(lo) <= abs(hi) * 2.0 ** -51, (i, r[:, i])


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not gpu_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("K", [2, 4, 8])
@pytest.mark.parametrize("kind", ["rand", "wide", "int"])
def test_add_mul_fma_vs_exact(K, kind):
    eps = Fraction(synth.EPS_P[K])
    n = N_RANDOM // (K // 2)
    a = _inputs(K, n, 10 + K, kind)
    b = _inputs(K, n, 20 + K, kind)
    c = _inputs(K, n, 30 + K, kind)
    # cancellation cases: b = -a + tiny for a quarter of the entries
    q = n // 4
    b[:, :q] = -a[:, :q]
    b[K - 1, :q] += a[0, :q] * 2.0 ** (-53 * K + 10)
    radd = _run(K, "add", a, b)
    rsub = _run(K, "sub", a, b)
    rmul = _run(K, "mul", a, b)
    rfma = _run(K, "fma", a, b, c.copy())
    worst = {"add": 0.0, "sub": 0.0, "mul": 0.0, "fma": 0.0}
    for i in range(n):
        fa, fb, fc = limbs_to_fraction(a[:, i]), limbs_to_fraction(b[:, i]), limbs_to_fraction(c[:, i])
        for name, r, exact, scale in (
            ("add", radd, fa + fb, abs(fa) + abs(fb)),
            ("sub", rsub, fa - fb, abs(fa) + abs(fb)),
            ("mul", rmul, fa * fb, abs(fa * fb)),
            ("fma", rfma, fc + fa * fb, abs(fc) + abs(fa * fb)),
        ):
            err = abs(limbs_to_fraction(r[:, i]) - exact)
            if scale == 0:
                assert err == 0
                continue
            worst[name] = max(worst[name], float(err / (eps * scale)))
    for r in (radd, rsub, rmul, rfma):
        _check_nonoverlap(r)
    # c_K, derived a priori from md.cuh (DESIGN R32), in units of u_K = 2^(-53K):
    #   K - 1 dropped products of level K, one rounding of the last output limb, and
    #   N_K = (K-2)(K+1) + K plain additions into the last level s[K-1] (every
    #   level_insert of prod_levels and of acc ends in one), each rounding a partial
    #   sum |s[K-1]| <= 4 u_{K-1} scale, i.e. an error <= 2 u_K scale:
    #   c_K = (K + 2 N_K) u_K / eps_p  ->  2d 1.5, 4d 8, 8d 66
    # (measured on B200: 0.74, 2.04, 37).  od keeps ~2^-417 relative (1e-120 needs 2^-399).
    print(f'md_worst K={K}', worst)
    u = {2: 2.0 ** -106, 4: 2.0 ** -212, 8: 2.0 ** -424}[K]
    c_k = (K + 2 * ((K - 2) * (K + 1) + K)) * u / synth.EPS_P[K]
    assert max(worst.values()) <= c_k, (c_k, worst)


@pytest.mark.parametrize("K", [2, 4, 8])
def test_div_sqrt_vs_exact(K):
    eps = Fraction(synth.EPS_P[K])
    n = 500
    a = np.abs(_inputs(K, n, 40 + K, "rand")) * 1.0
    a = _inputs(K, n, 41 + K, "rand")
    a[:, :] = np.where(a[0:1, :] < 0, -a, a)   # make every value positive
    b = _inputs(K, n, 42 + K, "rand")
    rdiv = _run(K, "div", a, b)
    rsq = _run(K, "sqrt", a)
    wd = ws = 0.0
    for i in range(n):
        fa, fb = limbs_to_fraction(a[:, i]), limbs_to_fraction(b[:, i])
        q = fa / fb
        wd = max(wd, float(abs(limbs_to_fraction(rdiv[:, i]) - q) / (eps * abs(q))))
        r = limbs_to_fraction(rsq[:, i])
        # |r - sqrt(a)| ~ |r^2 - a| / (2 sqrt a)
        ws = max(ws, float(abs(r * r - fa) / (2 * r * r) / eps))
    _check_nonoverlap(rdiv)
    _check_nonoverlap(rsq)
    print(f'md_divsqrt K={K}', wd, ws)
    assert wd <= {2: 8, 4: 16, 8: 64}[K] and ws <= {2: 8, 4: 16, 8: 64}[K], (wd, ws)


@pytest.mark.parametrize("K", [2, 4, 8])
def test_special_values(K):
    z = np.zeros((K, 6))
    a = z.copy(); b = z.copy()
    a[0] = [1.0, 0.0, 3.0, -2.0, 2.0 ** 53, 4.0]
    b[0] = [2.0 ** -60, 5.0, -3.0, 0.0, 1.0, 0.0]
    r = _run(K, "add", a, b)
    assert r[0, 0] == 1.0 and r[1, 0] == 2.0 ** -60
    assert r[0, 2] == 0.0 and not r[:, 2].any()              # x + (-x) = 0
    assert r[0, 4] == 2.0 ** 53 and r[1, 4] == 1.0           # S:49 two_sum case
    m = _run(K, "mul", a, b)
    assert m[0, 1] == 0.0 and m[0, 3] == 0.0                 # 0 * x
    s = _run(K, "sqrt", a)
    assert s[0, 5] == 2.0 and not s[1:, 5].any()             # sqrt(4) = 2 exactly
    assert not s[:, 1].any()                                 # sqrt(0) = 0


@pytest.mark.parametrize("K", [2, 4, 8])
def test_truncation_agrees_with_lower_precision(K):
    """a 4d result truncated to 2 limbs agrees with the 2d result to ~eps_2d."""
    if K == 2:
        pytest.skip("no lower precision")
    n = 300
    a = _inputs(K, n, 50, "rand")
    b = _inputs(K, n, 51, "rand")
    hi = _run(K, "mul", a, b)
    a2 = np.stack([synth.rational_to_md(*limbs_to_fraction(a[:, i]).as_integer_ratio(), 2) for i in range(n)], 1)
    b2 = np.stack([synth.rational_to_md(*limbs_to_fraction(b[:, i]).as_integer_ratio(), 2) for i in range(n)], 1)
    lo = _run(2, "mul", a2, b2)
    for i in range(n):
        h = limbs_to_fraction(hi[:2, i])
        l = limbs_to_fraction(lo[:, i])
        assert abs(h - l) <= abs(h) * Fraction(2) ** -100


def test_deterministic_runs():
    a = _inputs(8, 256, 60, "rand")
    b = _inputs(8, 256, 61, "rand")
    r1 = _run(8, "fma", a, b, a.copy())
    r2 = _run(8, "fma", a, b, a.copy())
    assert np.array_equal(r1, r2)
