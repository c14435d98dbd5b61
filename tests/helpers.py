"""Shared helpers for the GPU parity tests: run the oracle, convert GPU limbs to
exact values, and measure errors in units of the tolerance tol_p * s."""
from __future__ import annotations

from fractions import Fraction

import math

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
    """|gpu - oracle| / scale as a float (scale > 0).  mp fields: the limbs
    summed exactly in the field's precision (>= 2x the md bits, so the sum of
    K nonoverlapping doubles is exact), the difference in the field.  A
    non-finite GPU limb is an infinite error (max() would drop a NaN ratio)."""
    if not all(math.isfinite(float(l)) for l in gpu_limbs):
        return float("inf")
    if hasattr(F, "ctx") and not getattr(F, "is_complex", False):
        c = F.ctx
        g = c.fsum([c.mpf(float(l)) for l in gpu_limbs])
        diff = abs(g - oracle_val)
        if scale <= 0:
            return 0.0 if diff == 0 else float("inf")
        return float(diff) / scale
    diff = abs(limbs_to_fraction(gpu_limbs) - to_frac(F, oracle_val))
    if scale <= 0:
        return 0.0 if diff == 0 else float("inf")
    return float(diff / Fraction(scale))


def system_tensors(sys_, x_np, device="cuda:0"):
    import torch
    return torch.tensor(x_np, dtype=torch.float64, device=device).contiguous()


def eval_diff_errors(sys_, x_np, b_gpu, A_gpu, rows, F, pattern, oracle_bA=None):
    """max over sampled rows of |gpu - oracle| / (tol_p s) for b and A
    (oracle_bA: the oracle's (b, A) computed elsewhere, e.g. parallel_step)."""
    rp, ci = pattern
    K, d = sys_.K, sys_.d
    tol = synth.TOL_P[K]
    if oracle_bA is None:
        b, A = O.evaluate(sys_, O.read_x(x_np, F), F, split=True, rows=rows)
    else:
        b, A = oracle_bA
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
    """dx parity: max_k max_i |gpu - oracle| / (tol_p s_k); also per k the
    error in units of eps_p |x_k| (|x_k| = max_i |oracle x_new k,i|)."""
    n, d, K = sys_.n, sys_.d, sys_.K
    sc = O.scales(sys_, x_np)
    dxf = np.array([[float(out["dx"][k][i]) for i in range(n)] for k in range(d)])
    s_k, _ = O.stage_scales(sys_, x_np, dense_A0_float(out["A"], n), dxf, sc["s_b"], sc["s_A"])
    tol = synth.TOL_P[K]
    worst = 0.0
    worst_eps = 0.0
    per_k_eps_x = []
    for k in range(d):
        xk = max(abs(float(out["x_new"][i][k])) for i in range(n)) or 1.0
        wk = 0.0
        for i in range(n):
            r = err_ratio(dx_gpu[:, k, i], out["dx"][k][i], F, s_k[k])
            worst = max(worst, r / tol)
            worst_eps = max(worst_eps, r / synth.EPS_P[K])
            wk = max(wk, r * float(s_k[k]) / (synth.EPS_P[K] * xk))
        per_k_eps_x.append(wk)
    return dict(dx=worst, dx_eps=worst_eps, s=s_k, per_k_eps_x=per_k_eps_x)


def xnew_errors(sys_, x_np, out, x_gpu, F, s_k):
    n, d, K = sys_.n, sys_.d, sys_.K
    tol = synth.TOL_P[K]
    worst = 0.0
    for j in range(n):
        for k in range(d):
            r = err_ratio(x_gpu[:, j, k], out["x_new"][j][k], F, s_k[k])
            worst = max(worst, r / tol)
    return worst


# ---------------------------------------------------------------------------
# the oracle at full size: the same plain definition (oracle/newton.py),
# mapped over equations in worker processes (test infrastructure only)
# ---------------------------------------------------------------------------
def _procs():
    import os
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except Exception:
        return os.cpu_count() or 1


def _pk(v):
    """field value -> picklable (mpf/mpc of a private context do not pickle)"""
    if hasattr(v, "_mpc_"):
        return ("c", v._mpc_)
    return v._mpf_ if hasattr(v, "_mpf_") else v


def _unpk(F, t):
    if isinstance(t, tuple) and len(t) == 2 and t[0] == "c":
        return F.ctx.make_mpc(t[1])
    return F.ctx.make_mpf(t) if hasattr(F, "ctx") else t


def _field(prec):
    """the worker's field: 0 exact, >0 real mp, <0 complex mp of -prec bits"""
    if prec == 0:
        return O.ExactField()
    return O.ComplexMPField(-prec) if prec < 0 else O.MPField(prec)


def _prec_code(F):
    if not hasattr(F, "ctx"):
        return 0
    return -F.ctx.prec if getattr(F, "is_complex", False) else F.ctx.prec


def _rows_worker(args):
    sys_, x_np, prec, rows, dc = args
    F = _field(prec)
    xs = O.read_x(x_np, F)
    co = O.read_coeffs(sys_, F)
    rhs = O.read_rhs(sys_, F)
    out = {}
    for i in rows:
        bi, Ai = O.evaluate_row(sys_, xs, co, rhs, i, dc, F, split=True)
        out[i] = ([_pk(v) for v in bi], {j: [_pk(v) for v in ser] for j, ser in Ai.items()})
    return out


def _unpack_rows(F, parts):
    b, A = {}, {}
    for part in parts:
        for i, (bi, Ai) in part.items():
            b[i] = [_unpk(F, v) for v in bi]
            A[i] = {j: [_unpk(F, v) for v in ser] for j, ser in Ai.items()}
    return b, A


_STAGE = {}


def _stage_init(A_part, n, prec):
    F = _field(prec)
    _STAGE["A"] = {i: {j: [_unpk(F, v) for v in ser] for j, ser in row.items()} for i, row in A_part.items()}
    _STAGE["n"] = n
    _STAGE["F"] = F


def _stage_worker(args):
    """(A_j dx_{k-j})_i, j = j_lo..k, for the rows of this worker's A part
    (O.matvec_sparse, the oracle's own matvec)."""
    k, j_lo, new = args
    A, n, F = _STAGE["A"], _STAGE["n"], _STAGE["F"]
    dxs = _STAGE.setdefault("dx", [])   # dx_0, dx_1, ... sent once each
    dxs.extend([[_unpk(F, v) for v in dk] for dk in new])
    out = {i: [] for i in A}
    for j in range(j_lo, k + 1):
        Av = O.matvec_sparse(A, j, dxs[k - j], n, F)
        for i in A:
            out[i].append(_pk(Av[i]))
    return out  # per row, the terms of j = j_lo..k (subtracted in that order, as O.solve does)


def parallel_step(sys_, x_np, F, procs=None):
    """O.step with its per-equation work spread over processes:
    eval/diff row by row (O.evaluate_row), the stage recursion of Eq.(4) with
    the sparse matvecs split by rows and the LU solves (O.lu_factor /
    O.lu_solve) in this process.  Same arithmetic in the same order per
    value as O.step, so the same results."""
    import multiprocessing as mp
    procs = procs or _procs()
    n, d = sys_.n, sys_.d
    prec = _prec_code(F)
    # forkserver, not fork: the pytest process has CUDA (and its threads)
    # initialised; a forked child can deadlock on a lock held at fork time
    # (it hung the C3 full-parity test once)
    ctx = mp.get_context("forkserver")
    # LPT-ish deal: row costs grow with the monomial sizes
    cost = [sum(int(sys_.mono_ptr[t + 1] - sys_.mono_ptr[t]) for t in O.eq_monomials(sys_, i)) for i in range(n)]
    order = sorted(range(n), key=lambda i: -cost[i])
    chunks = [order[p::procs] for p in range(procs) if order[p::procs]]
    with ctx.Pool(len(chunks)) as pool:
        parts = pool.map(_rows_worker, [(sys_, x_np, prec, c, d) for c in chunks])
    b, A = _unpack_rows(F, parts)
    # A_j = 0 for j >= 1 when every input coefficient above 0 vanishes ('start')
    LU, perm = O.lu_factor(O.dense_coeff(A, n, 0, F), F)
    Aparts = [{i: {j: [_pk(v) for v in ser] for j, ser in A[i].items()} for i in c} for c in chunks]
    dx = []
    pools = [ctx.Pool(1, initializer=_stage_init, initargs=(ap, n, prec)) for ap in Aparts]
    try:
        for k in range(d):
            rhs = [b[i][k] for i in range(n)]
            if k > 0:
                dxp = [[_pk(v) for v in dx[k - 1]]]
                res = [p.apply_async(_stage_worker, ((k, 1, dxp),)) for p in pools]
                for r in res:
                    for i, vs in r.get().items():
                        for v in vs:
                            rhs[i] = rhs[i] - _unpk(F, v)
            dx.append(O.lu_solve(LU, perm, rhs, F))
        # residual r_k = b_k - sum_{j=0}^{k} A_j dx_{k-j}
        r = []
        for k in range(d):
            rk = [b[i][k] for i in range(n)]
            dxp = [[_pk(v) for v in dx[d - 1]]] if k == 0 else []
            res = [p.apply_async(_stage_worker, ((k, 0, dxp),)) for p in pools]
            for rr in res:
                for i, vs in rr.get().items():
                    for v in vs:
                        rk[i] = rk[i] - _unpk(F, v)
            r.append(rk)
    finally:
        for p in pools:
            p.close()
            p.join()
    x = O.read_x(x_np, F)
    x_new = [[x[i][k] + dx[k][i] for k in range(d)] for i in range(n)]
    bk = [[b[i][k] for i in range(n)] for k in range(d)]
    return dict(x=x, b=b, A=A, dx=dx, r=r, x_new=x_new, norm_b=O.series_norm(bk), norm_r=O.series_norm(r),
                norm_dx=O.series_norm(dx))


def parallel_rows(sys_, x_np, F, rows, procs=None):
    """(b_i, A_i) of the listed equations, in worker processes."""
    import multiprocessing as mp
    procs = min(procs or _procs(), len(rows))
    prec = _prec_code(F)
    chunks = [rows[p::procs] for p in range(procs) if rows[p::procs]]
    with mp.get_context("forkserver").Pool(len(chunks)) as pool:
        parts = pool.map(_rows_worker, [(sys_, x_np, prec, c, sys_.d) for c in chunks])
    return _unpack_rows(F, parts)


def vacuity(out, s_k, tol):
    """Per k: tol s_k / max_i |dx_k,i| (< 1: a wrong dx_k would be caught)."""
    ratios = []
    for k, dk in enumerate(out["dx"]):
        m = max(abs(complex(v)) for v in dk)  # the modulus (complex systems too)
        ratios.append(float("inf") if m == 0 else tol * float(s_k[k]) / m)
    return ratios


# ---------------------------------------------------------------------------
# complex systems (NEXT-2): errors as the modulus of the difference
# ---------------------------------------------------------------------------
def cplx_fraction(gpu_c_limbs):
    """[2][K] limbs -> (re, im) exact Fractions"""
    return limbs_to_fraction(gpu_c_limbs[0]), limbs_to_fraction(gpu_c_limbs[1])


def cerr_ratio(gpu_c_limbs, oracle_val, F, scale: float) -> float:
    re, im = cplx_fraction(gpu_c_limbs)
    ore, oim = F.to_fraction(oracle_val)
    return float(np.hypot(float(re - ore), float(im - oim))) / scale


def dense_A0_complex(A, n):
    M = np.zeros((n, n), complex)
    for i, row in A.items():
        for j, ser in row.items():
            M[i, j] = complex(ser[0])
    return M
