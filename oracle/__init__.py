"""CPU oracle for one Newton step on truncated power series (arxiv 2301.12659).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import or call
anything under ``oracle/``.  The product path (``paper_2301_12659_b200``)
never imports it and shares no code with it; the only shared module is the
seeded input generator ``synth`` (which holds none of the method's
arithmetic).

The oracle computes the plain DEFINITION of what the method computes
(SURVEY.md 8(c) c.1), in exact rational arithmetic (``fractions.Fraction``)
or in mpmath at at least twice the bits of the md precision under test:

* ``newton.evaluate``   b_k,i = [t^k](r_i - sum_tau c_tau prod_{j in tau} x_j)
                        A_k[i][j] = [t^k] sum_{tau ∋ j} c_tau prod_{l in tau, l != j} x_l
* ``newton.solve``      block forward substitution of the lower-triangular block
                        Toeplitz system Eq.(4) with Gaussian elimination
                        on A_0 (deliberately not QR: the least-squares solution of the
                        square nonsingular system equals A_0^{-1} b, reading R14)
* ``newton.step``       x + dx and the norms ||b||, ||b - A dx||, ||dx||
* ``newton.scales``     the running-error scales s_k of SURVEY.md 8(c) c.4 that
                        define the tolerance ||gpu_k - oracle_k|| <= tol_p s_k
* ``newton.step_window`` one step on the stage window [k_lo, dc) (Eq.(11));
                        ``newton.staggered_orders`` the Eq.(10) schedule (NEXT-1)
* ``newton.fabry_ratio`` c_{D-1}/c_D (Theorem 1); ``newton.residual_norm_sampled``
                        the residual of selected equations (NEXT-4)
* ``paper``             values the paper prints (T1, T2, Eq.(13)-(16) counts)

Parity status per function is listed in DESIGN.md "Oracle pins".  Entries
of Q and R are "parity unpinned" (sign freedom, reading R13); they are only
checked through dx and |R_jj|.
"""
from . import newton, paper  # noqa: F401
