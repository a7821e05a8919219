import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def orc():
    import oracle_lib

    return oracle_lib.oracle()


@pytest.fixture(scope="session")
def reflib():
    import oracle_lib

    if not oracle_lib.ref_available():
        pytest.skip("oracle/_ref (reference sources) not built")
    return oracle_lib.ref()


@pytest.fixture(scope="session")
def gpu():
    """The product path on the B200. Fails loudly (no fallback) if the native
    library or the device is missing."""
    from paper_1210_1491_b200 import _native

    return _native.context(0)
