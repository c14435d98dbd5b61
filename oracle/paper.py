"""Values PAPER.md prints, and the exact count laws it states.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
from __future__ import annotations

# T1 (tabMPneed): k, 1/k! as printed, precision, eps as printed.
T1 = [
    (7, "2.0e-004", "double precision", "2.2e-16"),
    (15, "7.7e-013", "use double doubles", "4.9e-32"),   # true 1/15! = 7.6e-13 (reading R27)
    (23, "3.9e-023", "use double doubles", None),
    (31, "1.2e-034", "use quad doubles", "6.1e-64"),
    (47, "3.9e-060", "use octo doubles", "4.6e-128"),
    (63, "5.0e-088", "use octo doubles", None),
    (95, "9.7e-149", "need hexa doubles", "5.3e-256"),
    (127, "3.3e-214", "need hexa doubles", None),
]

# T2 (tabcostmd): double operations per md multiplication (+, -, *, total)
T2 = {2: (5, 9, 9, 23), 4: (99, 164, 73, 336), 8: (529, 954, 259, 1742)}

# Eq.(16) factors
INTENSITY_FACTORS = {2: 11.5, 4: 84.0, 8: 217.75}
GROWTH_FACTORS = (7.30, 2.59)  # 84/11.5, 217.75/84 as printed


def products_per_monomial(m: int) -> int:
    """Series products to evaluate and differentiate a product of m variables
    in the three-column reverse mode: (m-1) + (m-2) + (m-2) = 3m - 5 for m >= 3
    (Eq.(12)-(13)); m = 2 needs 1, m = 1 needs 0 (reading R7)."""
    if m <= 1:
        return 0
    if m == 2:
        return 1
    return 3 * m - 5


def reverse_mode_jobs(m: int):
    """The job list of Eq.(12), 1-based variable names:
    forward f_q = f_{q-1} * x_{q+1} (f_0 = x_1), backward g_q = g_{q-1} * x_{m-q}
    (g_0 = x_m), cross d/dx_j = f_{j-2} * g_{m-j-1}, j = 2..m-1."""
    if m < 3:
        return [], [], []
    fwd = [(f"f{q-1}" if q > 1 else "x1", f"x{q+1}") for q in range(1, m)]
    bwd = [(f"g{q-1}" if q > 1 else f"x{m}", f"x{m-q}") for q in range(1, m - 1)]
    cross = []
    for j in range(2, m):
        a = f"f{j-2}" if j - 2 >= 1 else "x1"
        bq = m - j - 1
        b = f"g{bq}" if bq >= 1 else f"x{m}"
        cross.append((j, a, b))
    return fwd, bwd, cross


def padded_products(d: int) -> int:
    """Coefficient products of one padded convolution: d^2."""
    return d * d


def triangular_products(d: int) -> int:
    """Coefficient products of one truncated convolution without padding:
    sum_{k<d} (k+1) = d(d+1)/2 (the nonzero terms of Eq.(14))."""
    return d * (d + 1) // 2
