import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libguardian.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def oracle_lib():
    import oracle
    oracle.build()
    return oracle


@pytest.fixture
def arenas():
    """Factory of VMM arenas on cuda:0, all destroyed at teardown."""
    import torch
    from paper_2401_09290_b200 import guardian as g
    made = []

    def make(nbytes):
        a = g.Arena(0, nbytes)
        made.append(a)
        return a

    yield make
    torch.cuda.synchronize()
    for a in made:
        a.close()
    torch.cuda.empty_cache()
