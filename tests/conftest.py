import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def lr():
    import paper_1609_09068_b200 as m
    m.lib()
    return m


@pytest.fixture(scope="session")
def oracle():
    from oracle_py import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle_py import Ref
    if not Ref.available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return Ref()


FIXTURE8 = [(0, 1), (0, 2), (1, 3), (2, 4), (2, 5), (1, 5), (4, 5), (6, 7), (3, 1), (7, 6), (1, 6)]


def random_graph(rng, n, p, loops=False):
    import numpy as np
    A = rng.random((n, n)) < p
    if not loops:
        np.fill_diagonal(A, False)
    s, d = np.nonzero(A)
    return s.astype("int32"), d.astype("int32")
