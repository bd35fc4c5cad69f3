import os
import sys

# Multi-threaded OpenBLAS is ~10x slower than one thread on the small, skinny
# LAPACK calls the oracle makes (measured on the container host); pin one thread.
for _v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, "1")

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libwlr.so")
    config.addinivalue_line("markers", "slow: long-running oracle case")

try:  # numpy may already be imported by a plugin; enforce the limit at runtime too
    from threadpoolctl import threadpool_limits

    _limits = threadpool_limits(limits=1)
except Exception:  # pragma: no cover
    _limits = None
