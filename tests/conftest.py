import os
import sys

# single-threaded BLAS in the test process: after the oracle's worker pools,
# OpenBLAS's threaded inverse of the 128 x 128 A_0 (stage_scales) deadlocked the
# process and hung the C3 full-parity tests (a fresh process inverts it in 1 ms)
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")
try:  # numpy may already be loaded by a plugin: limit the live BLAS pool too
    from threadpoolctl import threadpool_limits
    threadpool_limits(1)
except Exception:  # pragma: no cover
    pass

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running oracle case")
