import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running CPU check")


@pytest.fixture(scope="session")
def orc():
    from oracles import oracle
    return oracle()


@pytest.fixture(scope="session")
def ref():
    from oracles import reflib
    r = reflib()
    if r is None:
        pytest.skip("oracle/_ref (reference build) not present")
    return r


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1706_06844_b200 as fde
    fde.load_library()
    return torch.device("cuda:0")
