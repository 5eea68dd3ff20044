import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")
REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: larger parity sweeps")


def have_reference() -> bool:
    return os.path.isdir(os.path.join(REFERENCE_SRC, "deltasnap"))


REFERENCE_INSTALL = os.path.join(ROOT, "baseline", "_ref")


def reference_path():
    """Where the unmodified reference package can be imported from: the
    offline pip install under baseline/_ref (travels to the GPU box), else the
    read-only source tree (build container only); None if neither exists."""
    for p in (REFERENCE_INSTALL, REFERENCE_SRC):
        if os.path.isdir(os.path.join(p, "deltasnap")):
            return p
    return None


def import_reference_anywhere():
    p = reference_path()
    if p is None:
        pytest.skip("the reference package is not installed (baseline/_ref)")
    sys.dont_write_bytecode = True
    if p not in sys.path:
        sys.path.insert(0, p)
    import deltasnap
    return deltasnap


def import_reference():
    """Import the reference package read-only (build container only)."""
    sys.dont_write_bytecode = True
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)
    import deltasnap
    return deltasnap


@pytest.fixture(scope="session")
def golden():
    import numpy as np

    cache = {}

    def load(name):
        if name not in cache:
            cache[name] = np.load(os.path.join(GOLDEN, f"{name}.npz"))
        return cache[name]

    return load
