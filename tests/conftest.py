import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200); runs through libsofg.so")
    config.addinivalue_line("markers", "slow: long-running")


def _has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def oracle():
    import oracle_lib

    return oracle_lib.get("reference") if oracle_lib.have_reference() else oracle_lib.get("port")


@pytest.fixture(scope="session")
def port():
    import oracle_lib

    return oracle_lib.get("port")


@pytest.fixture(scope="session")
def gpu_ctx():
    if not _has_gpu():
        pytest.fail("GPU test selected but no CUDA device is visible")
    import paper_2603_00326_b200 as sofg

    ctx = sofg.Context(0)
    yield ctx
    ctx.close()
