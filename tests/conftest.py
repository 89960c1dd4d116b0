import sys
from pathlib import Path
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs an sm_100 GPU (run with -m gpu on a B200)")


@pytest.fixture(scope="session")
def oracle():
    from oracle.bindings import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle.bindings import REF_SO, Ref
    if not REF_SO.exists():
        pytest.skip("reference build oracle/_ref/libssref.so not present")
    return Ref()


@pytest.fixture(scope="session")
def gpu_ctx():
    from paper_2505_08124_b200._lib import Context
    return Context(0)
