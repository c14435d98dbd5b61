"""Work accounting for one Newton step: exact md-operation
counts per kernel class from the system structure, and the static FP64
instruction mix of this library's md routines (counted from csrc/md.cuh; the
ncu cross-check is in profiles/).  Host-side bookkeeping only.

Numerators (always labelled):
  md_fma      algorithmic md multiply-adds (triangular convolutions, no padding)
  fp64_flops  md_fma x (DADD + DMUL + 2 DFMA) of our md_fma   -> "FP64 GFLOPS"
  fp64_instr  md_fma x (DADD + DMUL + DFMA) instructions      -> FP64-pipe fraction
  paper_flops md_mul x T2 cost (23/336/1742), context only (non-FMA counts)
"""
from __future__ import annotations

# FP64 instructions of one md fused accumulate r = acc + a*b (csrc/md.cuh fma_acc:
# product level sums, then acc inserted, then renorm)
#   K=2: two_prod (DMUL+DFMA) + 2 DFMA + two_sum (6) + 2 DADD + fast_two_sum (3)
#   K=4: product 9 two_sum + 10 DADD, acc 6 two_sum + 4 DADD, renorm 6 two_sum;
#        6 two_prod + 4 DFMA                               -> 140 DADD, 6 DMUL, 10 DFMA
#   K=8: product 127 two_sum + 54 DADD, acc 28 two_sum + 8 DADD, renorm 14 two_sum;
#        28 two_prod + 8 DFMA                              -> 1076 DADD, 28 DMUL, 36 DFMA
MD_FMA_MIX = {
    2: dict(dadd=11, dmul=1, dfma=3),
    4: dict(dadd=21 * 6 + 14, dmul=6, dfma=6 + 4),
    8: dict(dadd=169 * 6 + 62, dmul=28, dfma=28 + 8),
}
# md add: K(K-1)/2 cascade two_sum + K DADD + renorm 2(K-1) two_sum (K=2 specialised: 11)
MD_ADD_MIX = {2: dict(dadd=11, dmul=0, dfma=0),
              4: dict(dadd=12 * 6 + 4, dmul=0, dfma=0),
              8: dict(dadd=42 * 6 + 8, dmul=0, dfma=0)}
T2_MUL = {2: 23, 4: 336, 8: 1742}


def mix_flops(m):
    return m["dadd"] + m["dmul"] + 2 * m["dfma"]


def mix_instr(m):
    return m["dadd"] + m["dmul"] + m["dfma"]


def products(m: int) -> int:
    return 0 if m <= 1 else (1 if m == 2 else 3 * m - 5)


def step_counts(eq_ptr, mono_ptr, nnz: int, n: int, d: int, TB: int = 32) -> dict:
    """md multiply-adds per kernel class of one step (all orders 0..D)."""
    M = len(mono_ptr) - 1
    S = sum(products(int(mono_ptr[t + 1] - mono_ptr[t])) for t in range(M))
    conv = S * d * (d + 1) // 2                        # a2-a4: triangular convolutions
    scale = (M + sum(int(mono_ptr[t + 1] - mono_ptr[t]) for t in range(M))) * d   # a5
    qr = sum((n - j) + 2 * (2 * n - j - 1) * (n - j) for j in range(n))           # a6 on [A0 | I]
    updates = nnz * d * (d - 1) // 2                     # a7
    qhb = n * n * d                                      # a8 (explicit Q^T)
    T = (n + TB - 1) // TB
    bs = 0
    for t in range(T):                                   # a9 per stage
        t0, t1 = t * TB, min(n, (t + 1) * TB)
        bs += (t1 - t0) * (n - t1) + (t1 - t0) * (t1 - t0)
    bs *= d
    resid = n * n * d                                    # a10 dense A0 dx_k
    return dict(convolution=conv + scale, conv_products=conv, qr=qr, updates=updates, qhb=qhb, bs=bs,
                stage=updates + qhb + bs, residual=resid, series_products=S)


def algorithmic_counts(eq_ptr, mono_ptr, nnz: int, n: int, d: int) -> dict:
    """The method's work per kernel class of one step (all orders 0..D), in md
    multiply-adds, as SURVEY.md 8(a)/8(d) d.4 counts it -- independent of this
    implementation's formulation (which factors [A0 | I] and forms
    M = R^-1 Q^T once, so its own work differs):
      evaldiff  S d(d+1)/2 triangular convolutions (3m-5 per monomial, no
                padding) + (M + sum m) d coefficient scalings      (a2-a5)
      qr        (2/3) n^3 Householder QR of A_0                     (a6)
      stage     nnz d(d-1)/2 updates + 2 n^2 d for Q^T b (reflectors)
                + n^2 d / 2 back substitution                      (a7-a9)
      residual  nnz(A_0) d, the cheap form b'_k - A_0 dx_k           (a10)
    """
    M = len(mono_ptr) - 1
    ms = [int(mono_ptr[t + 1] - mono_ptr[t]) for t in range(M)]
    S = sum(products(m) for m in ms)
    evaldiff = S * d * (d + 1) // 2 + (M + sum(ms)) * d
    qr = (2 * n ** 3) // 3
    updates = nnz * d * (d - 1) // 2
    qhb = 2 * n * n * d
    bs = n * n * d // 2
    stage = updates + qhb + bs
    residual = nnz * d
    return dict(evaldiff=evaldiff, qr=qr, stage=stage, residual=residual, updates=updates, qhb=qhb, bs=bs,
                series_products=S, total=evaldiff + qr + stage + residual)


def flops(md_fma: int, K: int) -> int:
    return md_fma * mix_flops(MD_FMA_MIX[K])


def instr(md_fma: int, K: int) -> int:
    return md_fma * mix_instr(MD_FMA_MIX[K])


def fp64_peak_gflops(sm_count: int = 148, mhz: float = 1965.0) -> dict:
    """Derived FP64 peak (B200_PROFILING.md: 148 SMs; 64 FP64 lanes/SM/clk;
    sm_max_mhz from MEASURED_PEAKS.json): FMA-counted flops and pipe instructions."""
    lanes = sm_count * 64
    return dict(gflops=lanes * 2 * mhz * 1e-3, ginstr=lanes * mhz * 1e-3)
