"""GPU parity of the staggered Newton driver:
the windowed step (ns_set_window) against ``oracle.newton.step_window``, and
ns_run_newton against the closed-form solution and against an oracle replay
of the same windows.  Through the C ABI; tolerance tol_p * s_k (SURVEY c.4)."""
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


def _scales(sys_, x_np, out, dc):
    n, d = sys_.n, sys_.d
    sc = O.scales(sys_, x_np)
    dxf = np.zeros((d, n))
    for k in range(dc):
        dxf[k] = [float(v) for v in out["dx"][k]]
    A0 = np.zeros((n, n))
    for i, row in out["A"].items():
        for j, ser in row.items():
            A0[i, j] = float(ser[0])
    s_k, _ = O.stage_scales(sys_, x_np, A0, dxf, sc["s_b"], sc["s_A"])
    return s_k


@pytest.mark.parametrize("cfg,window", [("C1", (0, 1)), ("C1", (0, 4)), ("C1", (2, 9)), ("C1", (3, 7)),
                                        ("T4", (0, 5)), ("T4", (4, 16))])
def test_window_step_parity(cfg, window):
    import torch
    if cfg == "C1":
        sys_, F = synth.build_config("C1"), O.ExactField()
    else:
        sys_, F = synth.triangular_system(12, 15, 4, seed=7), O.MPField(512)
    k_lo, dc = window
    x_np = synth.make_x(sys_, "near", seed=3)
    h = _handle(sys_)
    h.set_window(k_lo, dc)
    x = torch.tensor(x_np, device="cuda:0")
    h.step(x)
    g = x.cpu().numpy()
    out = O.step_window(sys_, x_np, F, k_lo, dc, split=True)
    s_k = _scales(sys_, x_np, out, dc)
    tol = synth.TOL_P[sys_.K]
    worst = 0.0
    for j in range(sys_.n):
        for k in range(sys_.d):
            if k < k_lo or k >= dc:  # retired or outside the window: bitwise unchanged
                assert np.array_equal(g[:, j, k], x_np[:, j, k]), (j, k)
                continue
            worst = max(worst, H.err_ratio(g[:, j, k], out["x_new"][j][k], F, s_k[k]) / tol)
    assert worst <= 1.0, worst
    h.set_window(0, sys_.d)  # the full step again
    x2 = torch.tensor(x_np, device="cuda:0")
    h.step(x2)
    full = O.step(sys_, x_np, F, split=True)
    sf = _scales(sys_, x_np, full, sys_.d)
    w2 = max(H.err_ratio(x2.cpu().numpy()[:, j, k], full["x_new"][j][k], F, sf[k]) / tol
             for j in range(sys_.n) for k in range(sys_.d))
    assert w2 <= 1.0, w2


def _closed_form_errors(sys_, x_gpu, F):
    ex_np = synth.make_x(sys_, "exact")
    ex = O.read_x(ex_np, F)
    out = O.step(sys_, ex_np, F, split=True)  # the fixed point: dx ~ 0, gives A for the scales
    s_k = _scales(sys_, ex_np, out, sys_.d)
    tol = synth.TOL_P[sys_.K]
    return max(H.err_ratio(x_gpu[:, j, k], ex[j][k], F, s_k[k]) / tol
               for j in range(sys_.n) for k in range(sys_.d))


@pytest.mark.parametrize("cfg", ["C1", "T4"])
@pytest.mark.parametrize("qr_once", [False, True])
def test_run_newton_converges_to_closed_form(cfg, qr_once):
    import torch
    import paper_2301_12659_b200 as P
    if cfg == "C1":
        sys_, F = synth.build_config("C1"), O.MPField(256)
    else:
        sys_, F = synth.triangular_system(12, 15, 4, seed=7), O.MPField(512)
    x = torch.tensor(synth.make_x(sys_, "start", seed=5), device="cuda:0")
    h = _handle(sys_)
    info, log = h.run_newton(x, max_iter=24, flags=P.NS_QR_ONCE if qr_once else 0)
    assert info["converged"] == 1, (info, log)
    orders = O.staggered_orders(sys_.d)
    dcs = [e["dc"] for e in log]
    assert dcs[:len(orders)] == orders[:len(dcs)]
    assert all(v == sys_.d for v in dcs[len(orders):])
    klo = [e["k_lo"] for e in log]
    assert klo == sorted(klo) and info["k_lo"] == sys_.d
    assert info["qr_count"] == sum(e["qr"] for e in log)
    if qr_once:
        assert info["qr_count"] == 1
    else:  # refactored exactly while stage 0 was active
        assert all(e["qr"] == (1 if (e["k_lo"] == 0) else 0) for e in log)
    assert _closed_form_errors(sys_, x.cpu().numpy(), F) <= 1.0


def test_run_newton_replay_parity():
    """Replay the driver's windows (and its factorisation points) with the
    oracle from the same start: the final series agree element by element."""
    import torch
    sys_, F = synth.triangular_system(8, 15, 4, seed=11), O.MPField(512)
    x0 = synth.make_x(sys_, "start", seed=9)
    x = torch.tensor(x0, device="cuda:0")
    h = _handle(sys_)
    info, log = h.run_newton(x, max_iter=24)
    assert info["converged"] == 1
    xc = x0.copy()
    fact = None
    tol = synth.TOL_P[sys_.K]
    for e in log:
        if e["qr"]:
            fact = xc.copy()
        out = O.step_window(sys_, xc, F, e["k_lo"], e["dc"], split=True, x0_factor=fact)
        nxt = np.zeros((8,) + xc.shape[1:])
        for j in range(sys_.n):
            for k in range(sys_.d):
                v = F.to_fraction(out["x_new"][j][k])
                nxt[:, j, k] = synth.rational_to_md(v.numerator, v.denominator, 8)
        s_last = _scales(sys_, xc, out, e["dc"])
        xc = nxt[:sys_.K].copy()  # the oracle carries K limbs between iterations, like the GPU
    g = x.cpu().numpy()
    worst = max(H.err_ratio(g[:, j, k], F.num_fraction(H.limbs_to_fraction(xc[:, j, k])), F, s_last[k]) / tol
                for j in range(sys_.n) for k in range(sys_.d))
    assert worst <= 1.0, worst
