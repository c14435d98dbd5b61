"""-m "not gpu": the parallel driver of the oracle used by the full-size
parity tests (tests/helpers.parallel_step) gives exactly O.step's results."""
import synth
from oracle import newton as O
from tests import helpers as H


def test_parallel_step_equals_oracle_step():
    for sys_, kind in ((synth.triangular_system(9, 6, 4, seed=3), "rough"),
                       (synth.banded_two_column_system(10, 3, 5, 2, seed=4), "start")):
        x = synth.make_x(sys_, kind, seed=2)
        F = O.field_for(sys_.K)
        a = O.step(sys_, x, F, split=True)
        b = H.parallel_step(sys_, x, F, procs=3)
        for key in ("dx", "r", "x_new"):
            assert a[key] == b[key], key
        assert a["b"] == b["b"] and a["A"] == b["A"]
        assert a["norm_r"] == b["norm_r"] and a["norm_dx"] == b["norm_dx"]
        rb, rA = H.parallel_rows(sys_, x, F, [0, 4, 7], procs=2)
        assert all(rb[i] == a["b"][i] and rA[i] == a["A"][i] for i in (0, 4, 7))
