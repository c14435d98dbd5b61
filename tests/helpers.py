"""Shared helpers for the GPU parity tests: run the oracle, convert GPU limbs to
exact values, and measure errors in units of the tolerance tol_p * s."""
from __future__ import annotations

from fractions import Fraction

import numpy as np

import synth
from oracle import newton as O


def gpu_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def limbs_to_fraction(limbs) -> Fraction:
    s = Fraction(0)
    for l in limbs:
        s += Fraction(float(l))
    return s


def to_frac(F, v) -> Fraction:
    return F.to_fraction(v) if not isinstance(v, Fraction) else v


def err_ratio(gpu_limbs, oracle_val, F, scale: float) -> float:
    """|gpu - oracle| / scale as a float (scale > 0)."""
    diff = abs(limbs_to_fraction(gpu_limbs) - to_frac(F, oracle_val))
    if scale <= 0:
        return 0.0 if diff == 0 else float("inf")
    return float(diff / Fraction(scale))


def system_tensors(sys_, x_np, device="cuda:0"):
    import torch
    return torch.tensor(x_np, dtype=torch.float64, device=device).contiguous()


def eval_diff_errors(sys_, x_np, b_gpu, A_gpu, rows, F, pattern):
    """max over sampled rows of |gpu - oracle| / (tol_p s) for b and A."""
    rp, ci = pattern
    K, d = sys_.K, sys_.d
    tol = synth.TOL_P[K]
    xs = O.read_x(x_np, F)
    b, A = O.evaluate(sys_, xs, F, split=True, rows=rows)
    sc = O.scales(sys_, x_np)
    worst_b = worst_A = 0.0
    worst_b_eps = worst_A_eps = 0.0
    eps = synth.EPS_P[K]
    for i in rows:
        for k in range(d):
            s = max(sc["s_b"][k, i], 1e-300)
            r = err_ratio(b_gpu[:, k, i], b[i][k], F, s)
            worst_b = max(worst_b, r / tol)
            worst_b_eps = max(worst_b_eps, r / eps)
        for e in range(rp[i], rp[i + 1]):
            j = int(ci[e])
            ser = A[i].get(j)
            for k in range(d):
                s = max(sc["s_A"][(i, j)][k], 1e-300)
                r = err_ratio(A_gpu[:, k, e], ser[k], F, s)
                worst_A = max(worst_A, r / tol)
                worst_A_eps = max(worst_A_eps, r / eps)
    return dict(b=worst_b, A=worst_A, b_eps=worst_b_eps, A_eps=worst_A_eps)


def step_oracle(sys_, x_np, F):
    return O.step(sys_, x_np, F, split=True)


def dense_A0_float(A, n):
    M = np.zeros((n, n))
    for i, row in A.items():
        for j, ser in row.items():
            M[i, j] = float(ser[0])
    return M


def solve_errors(sys_, x_np, out, dx_gpu, F):
    """dx parity: max_k max_i |gpu - oracle| / (tol_p s_k)."""
    n, d, K = sys_.n, sys_.d, sys_.K
    sc = O.scales(sys_, x_np)
    dxf = np.array([[float(out["dx"][k][i]) for i in range(n)] for k in range(d)])
    s_k, _ = O.stage_scales(sys_, x_np, dense_A0_float(out["A"], n), dxf, sc["s_b"], sc["s_A"])
    tol = synth.TOL_P[K]
    worst = 0.0
    worst_eps = 0.0
    for k in range(d):
        for i in range(n):
            r = err_ratio(dx_gpu[:, k, i], out["dx"][k][i], F, s_k[k])
            worst = max(worst, r / tol)
            worst_eps = max(worst_eps, r / synth.EPS_P[K])
    return dict(dx=worst, dx_eps=worst_eps, s=s_k)


def xnew_errors(sys_, x_np, out, x_gpu, F, s_k):
    n, d, K = sys_.n, sys_.d, sys_.K
    tol = synth.TOL_P[K]
    worst = 0.0
    for j in range(n):
        for k in range(d):
            r = err_ratio(x_gpu[:, j, k], out["x_new"][j][k], F, s_k[k])
            worst = max(worst, r / tol)
    return worst
