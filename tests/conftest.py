import os
import pathlib
import sys

import numpy as np
import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
GOLDEN = pathlib.Path(__file__).resolve().parent / "golden" / "golden.npz"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: large-size GPU property tests")


@pytest.fixture(scope="session")
def golden():
    return dict(np.load(GOLDEN))


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import Reference, reference_available
    if not reference_available():
        pytest.skip("oracle/_ref/libmpkref.so not built (no /root/reference at build time)")
    return Reference()


@pytest.fixture(scope="session")
def ctx():
    import paper_2309_02228_b200 as mpkg
    c = mpkg.Context(int(os.environ.get("MPKG_DEVICE", "0")))
    yield c
    c.close()


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def assert_bitwise(a, b, what=""):
    a, b = bits(a), bits(b)
    assert a.shape == b.shape, f"{what}: shape {a.shape} != {b.shape}"
    if not np.array_equal(a, b):
        idx = np.flatnonzero(a.ravel() != b.ravel())
        i = idx[0]
        raise AssertionError(f"{what}: {len(idx)} of {a.size} differ; first at {i}: "
                             f"{a.ravel()[i].view(np.float64)} vs {b.ravel()[i].view(np.float64)}")
