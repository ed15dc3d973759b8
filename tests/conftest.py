import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def port():
    from oracle.bindings import Oracle
    return Oracle("port")


@pytest.fixture(scope="session")
def ref():
    from oracle.bindings import Oracle, ref_available
    if not ref_available():
        pytest.skip("reference library oracle/_ref/libdetlsh_ref.so not built")
    return Oracle("reference")


@pytest.fixture(scope="session")
def gpu():
    import paper_2406_10938_b200 as D
    if D.device_count() < 1:
        pytest.fail("no CUDA device visible to libdetlsh_b200 (gpu tests must run on a B200)")
    return D


def gaussian(n, d, seed, scale=1.0):
    return (np.random.Generator(np.random.PCG64(seed)).normal(0, scale, (n, d))).astype(np.float32)


def lattice(n, d, seed, lo=-2, hi=2):
    return np.random.Generator(np.random.PCG64(seed)).integers(lo, hi + 1, (n, d)).astype(np.float32)
