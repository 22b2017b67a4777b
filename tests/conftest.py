import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: long-running CPU test")
    # The ABI tests load the in-tree library: build it (nvcc cross-compiles for
    # sm_100a without a GPU) if a fresh checkout has not been built yet.
    lib = os.path.join(ROOT, "paper_1008_1366_b200", "libidconv.so")
    if not os.path.exists(lib):
        from paper_1008_1366_b200 import _build
        _build.build()


@pytest.fixture(scope="session")
def rng():
    import numpy as np
    return np.random.default_rng(1008_1366)
