import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_sessionstart(session):
    """The parity tests compare against the oracle's streams: the library's seeded RNG mode (its
    default is OS entropy, include/blindmatch.h bm_rng_mode)."""
    try:
        from paper_2408_06167_b200 import bm
    except ImportError:      # library not built: the ABI tests report it
        return
    bm.bm_rng_mode(bm.RNG_SEEDED)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running (still part of the default suites)")


@pytest.fixture(scope="session")
def O():
    from oracle import oracle
    oracle.lib()
    return oracle
