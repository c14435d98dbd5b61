"""GPU parity of NEXT-4: residual sampling and the
Fabry ratio (Theorem 1), through the C ABI, against the oracle."""
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


def _handle(sys_):
    import paper_2301_12659_b200 as P
    return P.NewtonSystem.from_system(sys_)


@pytest.mark.parametrize("cfg", ["C1", "C2", "C3"])
def test_fabry_ratio_parity(cfg):
    import torch
    sys_ = synth.build_config(cfg)
    F = O.field_for(sys_.K)
    x_np = synth.make_x(sys_, "near", seed=4)
    h = _handle(sys_)
    z = h.fabry_ratio(torch.tensor(x_np, device="cuda:0")).cpu().numpy()
    xs = O.read_x(x_np, F)
    worst = 0.0
    for j in range(sys_.n):
        want = O.fabry_ratio(xs[j], F)
        err = abs(H.limbs_to_fraction(z[:, j]) - F.to_fraction(want)) / abs(F.to_fraction(want))
        worst = max(worst, float(err) / synth.EPS_P[sys_.K])
    assert worst <= 64.0, worst  # a correctly rounded-ish md division: a few eps_p


def test_fabry_ratio_exact_and_polynomial():
    """x_j = 1/(1 - t/rho_j) with dyadic rho: coefficients rho^-k are exact
    and so is z = rho (bitwise); a zero last coefficient gives +inf."""
    import torch
    sys_ = synth.build_config("C2")
    K, n, d = sys_.K, sys_.n, sys_.d
    x = np.zeros((K, n, d))
    rhos = [2.0 ** (j % 5 - 2) * (-1) ** j for j in range(n)]
    for j, rho in enumerate(rhos):
        x[0, j, :] = [rho ** -k for k in range(d)]
    x[0, 3, d - 1] = 0.0
    h = _handle(sys_)
    z = h.fabry_ratio(torch.tensor(x, device="cuda:0")).cpu().numpy()
    for j, rho in enumerate(rhos):
        if j == 3:
            assert np.isinf(z[0, j]) and z[0, j] > 0
        else:
            assert z[0, j] == rho and not z[1:, j].any()


@pytest.mark.parametrize("rows", [[0], [1, 5, 7], list(range(8))])
def test_residual_sampling(rows):
    """Sampling changes only the residual norm: x after the step is bitwise the
    full step's, the sampled ||r|| is at most the full one (sums of the same
    per-row values), and it is within the tolerance of the oracle's sampled
    norm (exact rational arithmetic)."""
    import torch
    sys_ = synth.build_config("C1")
    x_np = synth.make_x(sys_, "near", seed=6)
    h = _handle(sys_)
    xa = torch.tensor(x_np, device="cuda:0")
    ra = torch.zeros((sys_.K, 3), dtype=torch.float64, device="cuda:0")
    h.step(xa, ra)
    h.set_residual_sample(rows)
    xb = torch.tensor(x_np, device="cuda:0")
    rb = torch.zeros_like(ra)
    h.step(xb, rb)
    h.set_residual_sample(None)
    assert torch.equal(xa, xb)
    full, samp = ra.cpu().numpy(), rb.cpu().numpy()
    assert np.array_equal(full[:, 0], samp[:, 0]) and np.array_equal(full[:, 2], samp[:, 2])
    assert H.limbs_to_fraction(samp[:, 1]) <= H.limbs_to_fraction(full[:, 1])
    out = O.step(sys_, x_np, O.ExactField())
    want = O.residual_norm_sampled(out["r"], rows)  # exact: 0 (the solve is exact in Q)
    sc = O.scales(sys_, x_np)
    bound = Fraction(synth.TOL_P[sys_.K]) * Fraction(float(sc["s_b"].sum()))
    assert abs(H.limbs_to_fraction(samp[:, 1]) - want) <= bound
    if rows == list(range(8)):
        assert np.array_equal(full[:, 1], samp[:, 1])  # same rows, same order


@pytest.mark.parametrize("rows", [[3], [1, 5, 7], [6, 2]])
def test_residual_sampling_nonzero_residual(rows):
    """Non-vacuous sampling parity: a step with a stale factorisation
    (NS_REUSE_QR after factoring the A_0 of another x_0, the modified Newton
    of P:665-668) has r_k = b'_k - A_0 dx_k != 0 (row 0, x_0 = r_0, has the
    same A_0 row for every x and so a zero residual; it is not sampled alone),
    so the sampled norm
    depends on which equations are selected.  Against the oracle's
    step_window(x0_factor=...) residual on the same rows (exact rationals)."""
    import torch

    import paper_2301_12659_b200 as P
    sys_ = synth.build_config("C1")
    xf = synth.make_x(sys_, "rough", seed=31)
    x_np = synth.make_x(sys_, "rough", seed=32)
    h = _handle(sys_)
    h.step(torch.tensor(xf, device="cuda:0"))                    # caches the factors of A_0(xf)
    h.set_residual_sample(rows)
    x = torch.tensor(x_np, device="cuda:0")
    res = torch.zeros((sys_.K, 3), dtype=torch.float64, device="cuda:0")
    h.step(x, res, flags=P.NS_REUSE_QR)
    h.set_residual_sample(None)
    got = H.limbs_to_fraction(res.cpu().numpy()[:, 1])
    F = O.ExactField()
    out = O.step_window(sys_, x_np, F, 0, sys_.d, x0_factor=xf)
    want = O.residual_norm_sampled(out["r"], rows)
    others = [O.residual_norm_sampled(out["r"], [i]) for i in range(sys_.n)]
    # the residual is far above the tolerance, and different rows give different norms
    sc = O.scales(sys_, x_np)
    bound = Fraction(synth.TOL_P[sys_.K]) * Fraction(float(sc["s_b"].sum())) * sys_.n
    assert want > 1000 * bound and len(set(others)) > 1
    assert abs(got - want) <= bound, (float(got), float(want))
