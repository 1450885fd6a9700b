import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running check")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN_DIR, "golden.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_arrays():
    return dict(np.load(os.path.join(GOLDEN_DIR, "golden.npz")))


@pytest.fixture(scope="session")
def oracle():
    from oracle import load_oracle

    return load_oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle import load_ref, ref_available

    if not ref_available():
        pytest.skip("reference build oracle/_ref/libqmcref.so not present")
    return load_ref()


@pytest.fixture(scope="session")
def columns64(golden):
    """Built-in Joe-Kuo matrices built by the ORACLE from the golden rows."""
    from oracle import load_oracle, ptr

    o = load_oracle()
    rows = golden["direction_numbers"]
    import ctypes as C

    s = np.array([r[1] for r in rows], np.uint32)
    a = np.array([r[2] for r in rows], np.uint32)
    ms = [np.array(r[3], np.uint32) for r in rows]
    mp = (C.c_void_p * len(ms))(*[m.ctypes.data for m in ms])
    cols = np.zeros((64, 52), np.uint32)
    o.qo_build_matrices(64, ptr(s), ptr(a), C.cast(mp, C.c_void_p), ptr(cols))
    return cols
