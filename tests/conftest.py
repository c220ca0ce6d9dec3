import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path)")
    config.addinivalue_line("markers", "slow: longer CPU oracle runs")


@pytest.fixture(scope="session")
def built():
    """Compile the CUDA library and the CPU checkers (no-op when up to date)."""
    import __graft_entry__ as ge

    ge.build_lib()
    from oracle import bindings

    bindings.build(ref=True)
    return True


@pytest.fixture(scope="session")
def oracle(built):
    from oracle.bindings import Restatement

    return Restatement()


@pytest.fixture(scope="session")
def reference(built):
    from oracle.bindings import Reference, reference_available

    if not reference_available():
        pytest.skip("oracle/_ref (the compiled reference) is not present on this machine")
    return Reference()


@pytest.fixture(scope="session")
def gpu(built):
    import torch

    if not torch.cuda.is_available():
        pytest.fail("gpu test selected but no CUDA device is visible")
    import paper_2410_22205_b200 as lsr

    lsr.lib()
    return lsr


def load_golden(name):
    return dict(np.load(os.path.join(GOLDEN, name), allow_pickle=False))


def golden_grid(rec):
    return dict(dim=int(rec["dim"]), dims=[int(v) for v in rec["dims"]], origin=[float(v) for v in rec["origin"]],
                dx=float(rec["dx"]))


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.int64)


SL_CASES = ["circle2d", "hull2d", "sphere3d", "torus3d", "hull3d", "flat3d"]
