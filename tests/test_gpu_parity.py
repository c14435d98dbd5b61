"""GPU parity of the whole hot path against the oracle,
through the C ABI, on seeded synthetic inputs (synth).

Tolerance (north_star): |gpu - oracle| <= tol_p * s elementwise, tol_p = 1e-28
(2d), 1e-60 (4d), 1e-120 (8d), s the running-error scale of SURVEY 8(c) c.4.
The tests also report the error in units of eps_p (T1) and fail above 64 eps_p,
which flags a bug long before the tolerance would.
"""
import math
from fractions import Fraction

import numpy as np
import pytest

import synth
from oracle import newton as O
from tests import helpers as H

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not H.gpu_available():
        pytest.skip("no CUDA device")


def _torch():
    import torch
    return torch


def _handle(sys_, max_batch=1):
    import paper_2301_12659_b200 as P
    return P.NewtonSystem.from_system(sys_, max_batch=max_batch)


def _np(t):
    _torch().cuda.synchronize()
    return t.detach().cpu().numpy()


def _run_all(sys_, x_np):
    """eval/diff, solve of the GPU's own (b, A, A0), and one full step."""
    torch = _torch()
    h = _handle(sys_)
    x = torch.tensor(x_np, device="cuda:0")
    b, A, A0 = h.eval_diff(x)
    dx = h.toeplitz_solve(b, A, A0)
    rdiag = h.r_diag()
    x2 = x.clone()
    res = torch.zeros((sys_.K, 3), dtype=torch.float64, device="cuda:0")
    h.step(x2, res)
    st = h.status()
    return dict(h=h, b=_np(b), A=_np(A), A0=_np(A0), dx=_np(dx), x_new=_np(x2), res=_np(res),
                rdiag=_np(rdiag), status=st.status_bits, pattern=h.pattern())


def _full_parity(sys_, x_np, F, eps_cap=64.0, out=None, nonvacuous=False, nonvacuous_k=None):
    """The whole step against the oracle (out: its result, computed here if
    None).  nonvacuous: assert tol_p s_k < max_i |dx_k,i| at every k < nonvacuous_k
    (default: every k), i.e. a wrong dx_k (even dx_k = 0) would fail the
    tolerance; beyond it the late-coefficient condition kappa_k makes
    any check at tol_p s_k vacuous (DESIGN 8)."""
    g = _run_all(sys_, x_np)
    if out is None:
        out = H.step_oracle(sys_, x_np, F)
    n, d, K = sys_.n, sys_.d, sys_.K
    ed = H.eval_diff_errors(sys_, x_np, g["b"], g["A"], list(range(n)), F, g["pattern"],
                            oracle_bA=(out["b"], out["A"]))
    assert ed["b"] <= 1 and ed["A"] <= 1, ed
    assert ed["b_eps"] <= eps_cap and ed["A_eps"] <= eps_cap, ed
    # dense A0 = structural A_0 scattered
    rp, ci = g["pattern"]
    A0 = np.zeros_like(g["A0"])
    for i in range(n):
        for e in range(rp[i], rp[i + 1]):
            A0[:, i, ci[e]] = g["A"][:, 0, e]
    assert np.array_equal(A0, g["A0"])
    sv = H.solve_errors(sys_, x_np, out, g["dx"], F)
    print(f"\n{sys_.name} n={n} d={d} K={K}: max err/(tol s) dx {sv['dx']:.2e}; per-k max err/(eps_p |x_k|): "
          + " ".join(f"{v:.1e}" for v in sv["per_k_eps_x"]))
    assert sv["dx"] <= 1, sv["dx"]
    if nonvacuous:
        vac = H.vacuity(out, sv["s"], synth.TOL_P[K])[:nonvacuous_k]
        assert max(vac) < 1.0, ("vacuous check at k =", [k for k, v in enumerate(vac) if v >= 1], vac)
    assert sv["dx_eps"] <= eps_cap * n, sv["dx_eps"]
    xe = H.xnew_errors(sys_, x_np, out, g["x_new"], F, sv["s"])
    assert xe <= 1, xe
    # norms: ||b|| and ||dx|| against the oracle's, the residual is at rounding level
    # norms (max over k of vector 1-norms): errors scale with the summed scales
    tol = synth.TOL_P[K]
    sb = O.scales(sys_, x_np)["s_b"]
    nb = H.limbs_to_fraction(g["res"][:, 0])
    assert abs(nb - H.to_frac(F, out["norm_b"])) <= Fraction(tol) * Fraction(float(sb.sum(axis=1).max()))
    ndx = H.limbs_to_fraction(g["res"][:, 2])
    assert abs(ndx - H.to_frac(F, out["norm_dx"])) <= Fraction(tol) * Fraction(float(max(sv["s"]))) * n
    nr = float(H.limbs_to_fraction(g["res"][:, 1]))
    assert nr <= tol * float(max(sv["s"])) * n
    assert g["status"] == 0
    return g, out, ed, sv


# ------------------------------------------------------------------ small / medium, all precisions
def test_C1_exact_tier():
    sys_ = synth.build_config("C1")
    for kind in ("near", "start"):
        x = synth.make_x(sys_, kind, seed=3)
        _full_parity(sys_, x, O.ExactField())


@pytest.mark.parametrize("K,n,D,seed", [(2, 40, 15, 1), (4, 36, 20, 2), (8, 34, 24, 3)])
def test_medium_triangular(K, n, D, seed):
    """spans two BS tiles (32 + ragged tail) and long monomials."""
    sys_ = synth.triangular_system(n, D, K, seed=seed)
    x = synth.make_x(sys_, "near", seed=seed + 10)
    _full_parity(sys_, x, O.field_for(K))


def test_two_column_banded():
    sys_ = synth.banded_two_column_system(40, 8, 10, 4, seed=5)
    x = synth.make_x(sys_, "near", seed=6)
    _full_parity(sys_, x, O.field_for(4))


@pytest.mark.parametrize("K", [2, 4, 8])
def test_degenerate_shapes(K):
    """n = 1 (m = 1 monomials only), D = 0 (one coefficient), a 2-variable system."""
    for sys_ in (synth.triangular_system(1, 5, K, seed=1),
                 synth.triangular_system(5, 0, K, seed=2),
                 synth.custom_system([[[0, 1]], [[1]]], [1.0, 1.0], 4, K, [0.9, -0.95])):
        x = synth.make_x(sys_, "near", seed=4)
        _full_parity(sys_, x, O.field_for(K))


# ------------------------------------------------------------------ bit-exact pins
@pytest.mark.parametrize("K", [2, 4, 8])
def test_integer_system_bit_exact(K):
    """x_j = 1/(1-t) + integer perturbation: every b and A coefficient is an
    integer < 2^53, so the GPU must reproduce the exact values bit for bit."""
    sys_ = synth.inv1mt_system(8, 8, K, two_column=True)
    x = synth.make_x(sys_, "int", seed=7)
    g = _run_all(sys_, x)
    F = O.ExactField()
    b, A = O.evaluate(sys_, O.read_x(x, F), F)
    rp, ci = g["pattern"]
    for i in range(sys_.n):
        for k in range(sys_.d):
            assert b[i][k].denominator == 1 and abs(b[i][k]) < 2 ** 53
            assert g["b"][0, k, i] == float(b[i][k]) and not g["b"][1:, k, i].any()
            for e in range(rp[i], rp[i + 1]):
                v = A[i][int(ci[e])][k]
                assert g["A"][0, k, e] == float(v) and not g["A"][1:, k, e].any()


@pytest.mark.parametrize("K", [2, 4, 8])
def test_zero_rhs_gives_zero_update_bitwise(K):
    """Eq.(11): at the exact 1/(1-t) solution b = 0 exactly, so
    QR dx_k = 0 => dx = 0 bit for bit and x is unchanged."""
    sys_ = synth.inv1mt_system(6, 7, K)
    x = synth.make_x(sys_, "exact")
    g = _run_all(sys_, x)
    assert not g["b"].any()
    assert not g["dx"].any()
    assert np.array_equal(g["x_new"], x)


# ------------------------------------------------------------------ Newton behaviour
@pytest.mark.parametrize("K,n,D", [(2, 8, 8), (4, 8, 15), (8, 6, 31)])
def test_quadratic_convergence_to_closed_form(K, n, D):
    """Iterated GPU steps from 'start' (x_0 correct to half precision)
    converge to exp(alpha t): coefficient k carries delta^(2^i - k) after i steps
    (SURVEY c.3), so after ceil(log2(D+2)) + 1 steps every coefficient is within
    tol_p s_k of the closed form, s_k the running-error scale at the solution
    (SURVEY c.4); the number of correct leading coefficients grows each step."""
    torch = _torch()
    sys_ = synth.triangular_system(n, D, K, seed=11)
    exact = synth.make_x(sys_, "exact")
    F = O.ExactField() if K == 2 else O.field_for(K)
    out = O.step(sys_, exact, F, split=True)
    sc = O.scales(sys_, exact)
    s_k, _ = O.stage_scales(sys_, exact, H.dense_A0_float(out["A"], n), np.zeros((D + 1, n)),
                            sc["s_b"], sc["s_A"])
    x = torch.tensor(synth.make_x(sys_, "start", seed=12), device="cuda:0")
    h = _handle(sys_)
    tol = synth.TOL_P[K]
    steps = math.ceil(math.log2(D + 2)) + 1
    ngood_prev = -1
    for it in range(1, steps + 1):
        h.step(x)
        xn = _np(x)
        ok = []
        for k in range(D + 1):
            e = max(abs(H.limbs_to_fraction(xn[:, j, k]) - H.limbs_to_fraction(exact[:, j, k])) for j in range(n))
            ok.append(e <= Fraction(tol) * Fraction(float(s_k[k])))
        ngood = ok.index(False) if False in ok else D + 1
        assert ngood > ngood_prev or ngood == D + 1, (it, ngood, ngood_prev)
        ngood_prev = ngood
    assert ngood_prev == D + 1, ngood_prev


def test_fixed_point():
    """From the rounded exact solution the update is at rounding level: ||dx|| <= tol."""
    torch = _torch()
    for K, n, D in ((2, 8, 8), (4, 16, 15), (8, 8, 31)):
        sys_ = synth.triangular_system(n, D, K, seed=21)
        x = torch.tensor(synth.make_x(sys_, "exact"), device="cuda:0")
        res = torch.zeros((K, 3), dtype=torch.float64, device="cuda:0")
        _handle(sys_).step(x, res)
        r = _np(res)
        assert abs(r[0, 2]) <= synth.TOL_P[K] * n   # ||dx||, coefficients are O(1)


# ------------------------------------------------------------------ API semantics
def test_reuse_qr_and_ledger():
    import paper_2301_12659_b200 as P
    torch = _torch()
    sys_ = synth.triangular_system(16, 7, 4, seed=3)
    h = _handle(sys_)
    x = torch.tensor(synth.make_x(sys_, "start", seed=1), device="cuda:0")
    with pytest.raises(P.NSError) as ei:
        h.step(x, flags=P.NS_REUSE_QR)
    assert ei.value.code == 10                              # NS_ESTATE
    h.step(x, flags=P.NS_LEDGER)
    h.step(x, flags=P.NS_LEDGER | P.NS_REUSE_QR)
    led = h.ledger()
    assert led["steps"] == 2 and led["qr_count"] == 1      # "QR once"
    assert led["ms_convolution"] > 0 and led["ms_stage"] > 0
    # operation counts beside the times: the closed forms of SURVEY 8(d) d.4
    from paper_2301_12659_b200 import perfmodel as PM
    c = PM.algorithmic_counts(sys_.eq_ptr, sys_.mono_ptr, h.nnz, sys_.n, sys_.d)
    assert led["md_fma_convolution"] == 2 * c["evaldiff"] and led["md_fma_qr"] == c["qr"]
    assert led["md_fma_stage"] == 2 * c["stage"] and led["md_fma_residual"] == 2 * c["residual"]
    assert led["flops_per_md_fma"] == PM.mix_flops(PM.MD_FMA_MIX[4])
    assert led["fp64_flops"] == led["flops_per_md_fma"] * (2 * c["total"] - c["qr"])
    assert P.lib().ns_newton_series_step(h._h, 8, 16, 7, x.data_ptr(), None, 0, None) == 2   # NS_EPREC
    assert P.lib().ns_newton_series_step(h._h, 4, 15, 7, x.data_ptr(), None, 0, None) == 3   # NS_EDIM


def test_deterministic_step():
    torch = _torch()
    sys_ = synth.triangular_system(40, 15, 4, seed=9)
    x0 = synth.make_x(sys_, "near", seed=2)
    outs = []
    for _ in range(2):
        h = _handle(sys_)
        x = torch.tensor(x0, device="cuda:0")
        h.step(x)
        outs.append(_np(x))
    assert np.array_equal(outs[0], outs[1])


# ------------------------------------------------------------------ batched (C5 shape)
def test_batched_matches_oracle_and_is_batch_invariant():
    torch = _torch()
    K, n, D = 2, 32, 15
    base = synth.build_config("C5")
    B = 24
    paths = [synth.triangular_system(n, D, K, seed=12665 + p) for p in range(B)]
    xs = np.stack([synth.make_x(s, "near", seed=100 + p) for p, s in enumerate(paths)])
    rhs = np.stack([s.rhs for s in paths])
    h = _handle(base, max_batch=B)
    X = torch.tensor(xs, device="cuda:0")
    R = torch.tensor(rhs, device="cuda:0")
    res = torch.zeros((B, K, 3), dtype=torch.float64, device="cuda:0")
    h.step_batched(X, R, res)
    Xn = _np(X)
    # batch invariance: path 5 alone gives the same bits
    X1 = torch.tensor(xs[5:6], device="cuda:0")
    h.step_batched(X1, torch.tensor(rhs[5:6], device="cuda:0"))
    assert np.array_equal(_np(X1)[0], Xn[5])
    # oracle parity on sampled paths
    F = O.field_for(K)
    for p in (0, 5, B - 1):
        out = O.step(paths[p], xs[p], F, split=True)
        sc = O.scales(paths[p], xs[p])
        dxf = np.array([[float(out["dx"][k][i]) for i in range(n)] for k in range(D + 1)])
        s_k, _ = O.stage_scales(paths[p], xs[p], H.dense_A0_float(out["A"], n), dxf, sc["s_b"], sc["s_A"])
        assert H.xnew_errors(paths[p], xs[p], out, Xn[p], F, s_k) <= 1
        nb = H.limbs_to_fraction(_np(res)[p, :, 0])
        assert abs(nb - H.to_frac(F, out["norm_b"])) <= Fraction(synth.TOL_P[K]) * Fraction(
            float(sc["s_b"].sum(axis=1).max()))


# ------------------------------------------------------------------ full BASELINE sizes
@pytest.mark.slow
@pytest.mark.parametrize("kind", ["near", "start", "rough"])
def test_C2_full_parity(kind):
    """configs[1]: dim=64, degree 31, quad double -- the whole step against the
    full oracle.  'start' (x_0 to half precision, the rest 0) and
    'rough' (every coefficient perturbed by 2^-12) make dx large at every k,
    so the tolerance tol_p s_k is asserted to be below |dx_k| (non-vacuous);
    'near' (the timing input) is the near-converged case."""
    sys_ = synth.build_config("C2")
    x = synth.make_x(sys_, kind, seed=1)
    F = O.field_for(4)
    # 'rough' at degree 31: kappa_k pushes tol_p s_k above |dx_k| from k = 17 on
    _full_parity(sys_, x, F, out=H.parallel_step(sys_, x, F), nonvacuous=(kind != "near"),
                 nonvacuous_k=(17 if kind == "rough" else None))


@pytest.mark.slow
def test_C3_full_parity_start():
    """configs[2]: dim=128, degree 63, octo double, 'start' input: every
    output of the step (b, A, dense A0, dx, x_new, norms) against the full
    oracle (parallel_step: the oracle's own functions over worker processes),
    non-vacuous at every k."""
    sys_ = synth.build_config("C3")
    x = synth.make_x(sys_, "start", seed=1)
    F = O.field_for(8)
    _full_parity(sys_, x, F, out=H.parallel_step(sys_, x, F), nonvacuous=True)


@pytest.mark.slow
def test_C3_full_parity_rough():
    """configs[2] with every coefficient perturbed ('rough'): the updates
    A_j dx_{k-j}, j >= 1, are all nonzero, so the bulk right-looking updates
    and the stage chain are exercised at every k; full oracle, non-vacuous."""
    sys_ = synth.build_config("C3")
    x = synth.make_x(sys_, "rough", seed=1)
    F = O.field_for(8)
    # 'rough' at degree 63: kappa_k ~ 1e4 per k pushes tol_p s_k above |dx_k| from k = 31 on
    _full_parity(sys_, x, F, out=H.parallel_step(sys_, x, F), nonvacuous=True, nonvacuous_k=31)


@pytest.mark.slow
def test_C3_sampled_parity():
    """configs[2]: dim=128, degree 63, octo double.  Sampled rows of b and A
    against the oracle; |R_jj| against the Cholesky factor of A0^T A0 (unique,
    unlike Q and R); dx through the residual of the block system on sampled rows
    with the GPU's verified A and b, evaluated exactly."""
    sys_ = synth.build_config("C3")
    x = synth.make_x(sys_, "near", seed=1)
    g = _run_all(sys_, x)
    F = O.field_for(8)
    rows = [0, 1, 2, 63, 127]
    ed = H.eval_diff_errors(sys_, x, g["b"], g["A"], rows, F, g["pattern"])
    assert ed["b"] <= 1 and ed["A"] <= 1, ed
    n, d, K = sys_.n, sys_.d, 8
    # |R_jj| = diag of the Cholesky factor of A0^T A0
    A0 = [[F.from_limbs(g["A0"][:, i, j]) for j in range(n)] for i in range(n)]
    G = [[sum((A0[r][i] * A0[r][j] for r in range(n)), F.zero) for j in range(n)] for i in range(n)]
    L = F.ctx.cholesky(F.ctx.matrix(G))
    for j in range(n):
        rj = abs(H.limbs_to_fraction(g["rdiag"][:, j]))
        lj = H.to_frac(F, L[j, j])
        assert abs(rj - lj) <= Fraction(synth.TOL_P[K]) * lj * n
    # block-system residual of the GPU dx on sampled rows, exact arithmetic on
    # GPU A, b.  QR's backward error is normwise, so the scale is the max over
    # ALL rows of |b_k,i| + sum_j |A_j| |dx_{k-j}| (float64 magnitudes).
    rp, ci = g["pattern"]
    tol = synth.TOL_P[K]
    Aab = np.abs(g["A"][0])            # [d][nnz]
    dxab = np.abs(g["dx"][0])          # [d][n]
    bab = np.abs(g["b"][0])            # [d][n]
    for k in range(0, d, 7):
        rowscale = bab[k].copy()
        for j in range(k + 1):
            contrib = Aab[j] * dxab[k - j][ci]
            rowscale += np.add.reduceat(contrib, rp[:-1]) * (np.diff(rp) > 0)
        scale_k = Fraction(float(rowscale.max()))
        for i in (0, 64, 127):
            r = H.limbs_to_fraction(g["b"][:, k, i])
            for j in range(k + 1):
                for e in range(rp[i], rp[i + 1]):
                    r -= H.limbs_to_fraction(g["A"][:, j, e]) * H.limbs_to_fraction(g["dx"][:, k - j, ci[e]])
            assert abs(r) <= Fraction(tol) * scale_k, (i, k, float(abs(r) / scale_k))


@pytest.mark.parametrize("K,n,D", [(4, 36, 20), (8, 40, 12)])
def test_tiled_back_substitution_mode(K, n, D):
    """NS_TILED_BS: per stage y = Q^T b'_k then tiled back substitution (P:659-663,
    P:124-126) instead of dx_k = M b'_k; both must meet the tolerance."""
    import paper_2301_12659_b200 as P
    torch = _torch()
    sys_ = synth.triangular_system(n, D, K, seed=31)
    x_np = synth.make_x(sys_, "near", seed=32)
    F = O.field_for(K)
    out = H.step_oracle(sys_, x_np, F)
    sc = O.scales(sys_, x_np)
    dxf = np.array([[float(out["dx"][k][i]) for i in range(n)] for k in range(D + 1)])
    s_k, _ = O.stage_scales(sys_, x_np, H.dense_A0_float(out["A"], n), dxf, sc["s_b"], sc["s_A"])
    for flags in (P.NS_TILED_BS, 0):
        h = _handle(sys_)
        x = torch.tensor(x_np, device="cuda:0")
        h.step(x, flags=flags)
        assert H.xnew_errors(sys_, x_np, out, _np(x), F, s_k) <= 1, flags


def test_sharded_evaldiff_rows_bitwise_and_step_from():
    """C4 path on one GPU: eval/diff sharded over 3 equation ranges (three
    handles = three simulated ranks), rows assembled, must equal the unsharded
    eval/diff bit for bit (every row is computed by the same kernel code in
    the same order); the step from the assembled (b, A, A0) meets the tolerance."""
    from paper_2301_12659_b200.dist import equation_partition
    torch = _torch()
    sys_ = synth.banded_two_column_system(48, 6, 9, 4, seed=41)
    x_np = synth.make_x(sys_, "near", seed=42)
    x = torch.tensor(x_np, device="cuda:0")
    full = _handle(sys_)
    b, A, A0 = full.eval_diff(x)
    rp, ci = full.pattern()
    ranges = equation_partition(sys_.eq_ptr, sys_.mono_ptr, sys_.d, 3)
    bs, As, A0s = torch.zeros_like(b), torch.zeros_like(A), torch.zeros_like(A0)
    for lo, hi in ranges:
        h = _handle(sys_)
        h.set_partition(lo, hi)
        pb, pA, p0 = h.eval_diff(x)
        bs[:, :, lo:hi] = pb[:, :, lo:hi]
        As[:, :, rp[lo]:rp[hi]] = pA[:, :, rp[lo]:rp[hi]]
        A0s[:, lo:hi] = p0[:, lo:hi]
    assert torch.equal(bs, b) and torch.equal(As, A) and torch.equal(A0s, A0)
    F = O.field_for(4)
    out = H.step_oracle(sys_, x_np, F)
    sc = O.scales(sys_, x_np)
    n, D = sys_.n, sys_.D
    dxf = np.array([[float(out["dx"][k][i]) for i in range(n)] for k in range(D + 1)])
    s_k, _ = O.stage_scales(sys_, x_np, H.dense_A0_float(out["A"], n), dxf, sc["s_b"], sc["s_A"])
    x2 = x.clone()
    res = torch.zeros((4, 3), dtype=torch.float64, device="cuda:0")
    full.step_from(x2, bs, As, A0s, res)
    assert H.xnew_errors(sys_, x_np, out, _np(x2), F, s_k) <= 1


# ------------------------------------------------------------------ C4 shape and the large-n code paths
class _env:
    """environment overrides read by ns_system_create (launch-shape knobs)"""

    def __init__(self, **kw):
        self.kw = kw

    def __enter__(self):
        import os
        self.old = {k: os.environ.get(k) for k in self.kw}
        os.environ.update({k: str(v) for k, v in self.kw.items()})

    def __exit__(self, *a):
        import os
        for k, v in self.old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


@pytest.mark.slow
@pytest.mark.parametrize("split", [1, 0])
def test_n160_grid_qr_streaming_and_stage_paths(split):
    """n = 160 > 128: the grid QR's rows beyond its 32 S register window are
    streamed from L2, and (split = 0) the non-split stage_kernel that C4
    (n = 1024) runs; 2-column banded system with signed md coefficients
    (the C4 structure at w = 32), 'rough' input: full oracle parity."""
    # degree 12: at w = 32 the late-coefficient condition kappa_k grows ~1e4 per k,
    # beyond k ~ 13 tol_p s_k exceeds |dx_k| (a vacuous check, asserted against)
    sys_ = synth.banded_two_column_system(160, 32, 12, 4, seed=44)
    x = synth.make_x(sys_, "rough", seed=45)
    F = O.field_for(4)
    out = H.parallel_step(sys_, x, F)
    with _env(NS_STAGE_SPLIT=split):
        _full_parity(sys_, x, F, out=out, nonvacuous=True)


@pytest.mark.parametrize("K,bw", [(2, 16), (4, 32), (8, 128), (4, 128)])
def test_wy_solve_path(K, bw):
    """Blocked WY solve (wy.cuh; the default for n > 256): QR of A_0 alone,
    T_p = S_p^-1 per block of bw reflectors, per stage Q^T b'_k by blocks and
    back substitution by bw-row tiles.  Forced on at n = 40 (NS_WY=1): several
    blocks and a partial last block (bw = 16, 32), one identity-padded block
    (bw = 128); full oracle parity on 'rough' input."""
    # degree 7 at 2d: from k = 8 on tol_p s_k exceeds |dx_k| (a vacuous check)
    sys_ = synth.triangular_system(40, 7 if K == 2 else 12, K, seed=49)
    x = synth.make_x(sys_, "rough", seed=50)
    with _env(NS_WY=1, NS_WY_BW=bw):
        _full_parity(sys_, x, O.field_for(K), nonvacuous=True)


def test_wy_solve_path_n300_banded():
    """n = 300 > 256 takes the WY path by default: three blocks of 128 (the last
    partial), the 2-column banded structure of C4 with signed md coefficients."""
    sys_ = synth.banded_two_column_system(300, 8, 6, 4, seed=51)
    x = synth.make_x(sys_, "rough", seed=52)
    F = O.field_for(4)
    out = H.parallel_step(sys_, x, F)
    _full_parity(sys_, x, F, out=out, nonvacuous=True)


@pytest.mark.parametrize("K,env", [(8, dict(NS_QR_CRIT=1)), (4, dict(NS_QR_CRIT=1, NS_WY=1, NS_WY_BW=16)),
                                   (4, dict(NS_QR_INTERLEAVE=0)), (4, dict(NS_QR_INTERLEAVE=0, NS_WY=1))])
def test_grid_qr_variants(K, env):
    """The grid-QR variants: a dedicated critical-chain CTA (NS_QR_CRIT) on
    [A0 | I] and on A0 alone (the WY path), and the contiguous column ownership
    (NS_QR_INTERLEAVE=0) of both: full oracle parity on 'rough' input."""
    sys_ = synth.triangular_system(40, 12, K, seed=53)
    x = synth.make_x(sys_, "rough", seed=54)
    with _env(**env):
        _full_parity(sys_, x, O.field_for(K), nonvacuous=True)


@pytest.mark.parametrize("K,env", [(8, dict(NS_WYM=0)), (8, dict(NS_WYM=1)), (4, dict(NS_CQR=0, NS_WYM=1)),
                                   (4, dict(NS_CQR=0, NS_WYM=0)), (2, dict(NS_CQR=0, NS_WYM=1, NS_TILED_BS_ENV=1))])
def test_qr_of_a0_alone_and_qt_from_wy(K, env):
    """n <= 256 without the cluster QR: the QR of A_0 alone with Q^T = I - V T^T V^T
    formed from one WY block (NS_WYM=1, the default) against [A_0 | I] (NS_WYM=0);
    full oracle parity on 'rough' input (also the tiled back substitution on Q^T)."""
    import paper_2301_12659_b200 as P
    torch = _torch()
    sys_ = synth.triangular_system(40, 7 if K == 2 else 12, K, seed=55)
    x = synth.make_x(sys_, "rough", seed=56)
    F = O.field_for(K)
    env = dict(env)
    tiled = env.pop("NS_TILED_BS_ENV", 0)
    with _env(**env):
        if not tiled:
            _full_parity(sys_, x, F, nonvacuous=True)
            return
        out = H.step_oracle(sys_, x, F)
        sc = O.scales(sys_, x)
        n, d = sys_.n, sys_.d
        dxf = np.array([[float(out["dx"][k][i]) for i in range(n)] for k in range(d)])
        s_k, _ = O.stage_scales(sys_, x, H.dense_A0_float(out["A"], n), dxf, sc["s_b"], sc["s_A"])
        h = _handle(sys_)
        xt = torch.tensor(x, device="cuda:0")
        h.step(xt, flags=P.NS_TILED_BS)
        assert H.xnew_errors(sys_, x, out, _np(xt), F, s_k) <= 1


@pytest.mark.parametrize("owner", [0, 1])
def test_grid_qr_owner_beta_modes(owner):
    """NS_QR_OWNER_BETA: the reflector's owner forms beta (1, default) or each
    consumer forms it (0); both within tol_p s_k of the oracle."""
    sys_ = synth.triangular_system(40, 12, 8, seed=47)
    x = synth.make_x(sys_, "rough", seed=48)
    with _env(NS_QR_OWNER_BETA=owner):
        _full_parity(sys_, x, O.field_for(8), nonvacuous=True)


@pytest.mark.slow
def test_C4_sampled_rows_and_a_posteriori_residual():
    """configs[3] at full size (n = 1024, w = 32, degree 31, 4d), 'rough' input.
    (1) b and A on sampled equations against the oracle (SURVEY d.6);
    (2) the GPU dx solves the block system: on those equations the residual
    r_k,i = b_k,i - sum_{j<=k} (A_j dx_{k-j})_i, evaluated exactly on the
    GPU's verified A, b and its dx, is within tol_p times the normwise scale
    max_i' (|b_k| + sum_j |A_j| |dx_{k-j}|)_i' (Householder QR is normwise
    backward stable, reading R33), and that bound is far below |b_k| on those
    rows (a wrong dx, e.g. 0, fails); (3) the step's x_new = x + dx of the
    solve bit for bit."""
    sys_ = synth.build_config("C4")
    x = synth.make_x(sys_, "rough", seed=1)
    g = _run_all(sys_, x)
    F = O.field_for(4)
    rows = [0, 1, 31, 32, 500, 511, 512, 1022, 1023]
    ob, oA = H.parallel_rows(sys_, x, F, rows)
    ed = H.eval_diff_errors(sys_, x, g["b"], g["A"], rows, F, g["pattern"], oracle_bA=(ob, oA))
    assert ed["b"] <= 1 and ed["A"] <= 1, ed
    rp, ci = g["pattern"]
    K, d = 4, sys_.d
    tol = synth.TOL_P[K]
    Aab, dxab, bab = np.abs(g["A"][0]), np.abs(g["dx"][0]), np.abs(g["b"][0])
    worst = 0.0
    X = O.MPField(1400)  # the products of two 4d numbers and their sums, exact to far below tol_p
    val = lambda limbs: X.ctx.fsum([X.ctx.mpf(float(l)) for l in limbs])
    for k in range(d):
        rowscale = bab[k].copy()
        for j in range(k + 1):
            rowscale += np.add.reduceat(Aab[j] * dxab[k - j][ci], rp[:-1]) * (np.diff(rp) > 0)
        scale_k = float(rowscale.max())
        assert max(bab[k][i] for i in rows) > 1e6 * tol * scale_k  # non-vacuous
        for i in rows:
            r = val(g["b"][:, k, i])
            for j in range(k + 1):
                for e in range(rp[i], rp[i + 1]):
                    r -= val(g["A"][:, j, e]) * val(g["dx"][:, k - j, ci[e]])
            worst = max(worst, float(abs(r)) / scale_k / tol)
    print(f"\nC4 a-posteriori residual: max |r| / (tol_p scale) = {worst:.2e}")
    assert worst <= 1, worst
    # (3) the step's own update dx' = x_new - x (the step forms A_0 inside the QR
    # kernel, a0_row, so its dx is not bitwise the solve's): the same
    # a-posteriori residual check on the sampled equations
    xn = g["x_new"]
    worst2 = 0.0
    cols = sorted({int(ci[e]) for i in rows for e in range(rp[i], rp[i + 1])})
    dxs = {(c, k): val(xn[:, c, k]) - val(x[:, c, k]) for c in cols for k in range(d)}
    # x_new = x (+) dx is one md addition: |x_new - (x + dx)| <= 8 eps_p (|x| + |dx|)
    # (reading R32, c_4 <= 8), which A_j carries into the residual
    xdx = np.abs(x[0]).T + dxab  # [d][n]
    for k in range(d):
        rowscale = bab[k].copy()
        addb = np.zeros(sys_.n)
        for j in range(k + 1):
            rowscale += np.add.reduceat(Aab[j] * dxab[k - j][ci], rp[:-1]) * (np.diff(rp) > 0)
            addb += np.add.reduceat(Aab[j] * xdx[k - j][ci], rp[:-1]) * (np.diff(rp) > 0)
        scale_k = float(rowscale.max())
        for i in rows:
            r = val(g["b"][:, k, i])
            for j in range(k + 1):
                for e in range(rp[i], rp[i + 1]):
                    r -= val(g["A"][:, j, e]) * dxs[(int(ci[e]), k - j)]
            bound = tol * scale_k + 8 * synth.EPS_P[K] * float(addb[i])
            worst2 = max(worst2, float(abs(r)) / bound)
    print(f"C4 a-posteriori residual of the step's x_new - x: {worst2:.2e}")
    assert worst2 <= 1, worst2


def test_library_row_replication_kernels_bitwise():
    """The device half of the library's C4 exchange: three simulated ranks
    (ns_set_partition on three handles, ranges of ns_exchange_plan) pack their
    rows with ns_pack_rows into one gather buffer (what the grouped
    ncclBroadcast delivers to every rank), each unpacks the other blocks into
    its partial arrays: every rank then holds the unsharded eval/diff bitwise."""
    import paper_2301_12659_b200 as P
    torch = _torch()
    sys_ = synth.banded_two_column_system(48, 6, 9, 4, seed=41)
    x = torch.tensor(synth.make_x(sys_, "rough", seed=42), device="cuda:0")
    full = _handle(sys_)
    fb, fA, f0 = full.eval_diff(x)
    bounds, cnt = P.exchange_plan(sys_.eq_ptr, sys_.mono_ptr, sys_.var_idx, sys_.n, sys_.D, sys_.K, 3)
    off = np.concatenate([[0], np.cumsum(cnt)])
    gather = torch.zeros(int(off[-1]), dtype=torch.float64, device="cuda:0")
    parts = []
    for r in range(3):
        h = _handle(sys_)
        h.set_partition(int(bounds[r]), int(bounds[r + 1]))
        pb, pA, p0 = h.eval_diff(x)
        h.pack_rows(int(bounds[r]), int(bounds[r + 1]), pb, pA, p0, gather[off[r]:off[r + 1]])
        parts.append((h, pb, pA, p0))
    for r, (h, pb, pA, p0) in enumerate(parts):
        for q in range(3):
            if q != r:
                h.pack_rows(int(bounds[q]), int(bounds[q + 1]), pb, pA, p0, gather[off[q]:off[q + 1]], unpack=True)
        assert torch.equal(pb, fb) and torch.equal(pA, fA) and torch.equal(p0, f0), r


def test_library_nccl_comm_single_rank():
    """ns_nccl_unique_id + ns_comm_init on one rank (the library-owned NCCL
    communicator; one GPU here): the step through the sharded path equals the
    plain step bitwise and the communicator reports no asynchronous error."""
    import paper_2301_12659_b200 as P
    torch = _torch()
    sys_ = synth.banded_two_column_system(40, 6, 9, 4, seed=43)
    x_np = synth.make_x(sys_, "rough", seed=44)
    ref = _handle(sys_)
    xa = torch.tensor(x_np, device="cuda:0")
    ref.step(xa)
    h = _handle(sys_)
    h.comm_init(1, 0, P.nccl_unique_id())
    xb = torch.tensor(x_np, device="cuda:0")
    h.step(xb)
    torch.cuda.synchronize()
    assert torch.equal(xa, xb)
    assert h.comm_status() == 0


@pytest.mark.parametrize("K", [2, 4, 8])
def test_general_exponents(K):
    """NEXT-3 general exponents (reading R37): x_j^e written as e
    copies of j in a monomial, several monomials per equation; the single-
    system step and the batched kernel against the oracle, 'rough' input."""
    sys_ = synth.custom_system([[[0, 0, 1]], [[1, 1], [0]], [[0, 2, 2, 2]], [[1, 3, 3], [2]], [[0, 1, 2, 3, 4, 4]]],
                               [1.0, -0.5, 1.0, 0.75, 1.0, -0.25, 1.0], 9, K, [0.9, -0.95, 0.875, -1.0, 0.9375])
    x = synth.make_x(sys_, "rough", seed=7)
    F = O.field_for(K)
    _full_parity(sys_, x, F, nonvacuous=True)
    import torch
    h = _handle(sys_, max_batch=3)
    X = torch.tensor(np.stack([x] * 3), device="cuda:0")
    h.step_batched(X)
    out = O.step(sys_, x, F, split=True)
    sc = O.scales(sys_, x)
    n, D = sys_.n, sys_.D
    dxf = np.array([[float(out["dx"][k][i]) for i in range(n)] for k in range(D + 1)])
    s_k, _ = O.stage_scales(sys_, x, H.dense_A0_float(out["A"], n), dxf, sc["s_b"], sc["s_A"])
    assert H.xnew_errors(sys_, x, out, _np(X)[1], F, s_k) <= 1
