import glob
import os
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) GPU")


@pytest.fixture(scope="session")
def oracle_lib():
    import oracle

    return oracle.Oracle()


@pytest.fixture(scope="session")
def reference_lib():
    import oracle

    if not oracle.Reference.available():
        pytest.skip("oracle/_ref not built (reference tree absent when building)")
    return oracle.Reference()


@pytest.fixture(scope="session")
def ctx():
    import paper_2108_05021_b200 as ob

    c = ob.Context(0)
    yield c
    c.close()


def golden_cases():
    return sorted(p for p in glob.glob(os.path.join(GOLDEN_DIR, "*.npz"))
                  if not p.endswith("sat_2x2.npz"))


def fastosbf_golden_cases():
    return sorted(glob.glob(os.path.join(GOLDEN_DIR, "fastosbf", "*.npz")))


def boxfilter_golden_cases():
    return sorted(glob.glob(os.path.join(GOLDEN_DIR, "boxfilter", "*.npz")))


def filter3d_golden_cases():
    return sorted(glob.glob(os.path.join(GOLDEN_DIR, "filters3d", "*.npz")))


def smooth_golden_cases():
    return sorted(glob.glob(os.path.join(GOLDEN_DIR, "smooth", "*.npz")))


def load_golden(path):
    d = np.load(path)
    return {k: d[k] for k in d.files}


def bits(a):
    """View float64 data as uint64 for bit-exact comparisons."""
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)
