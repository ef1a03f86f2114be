import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through libfsvd_b200.so on cuda:0)")
    config.addinivalue_line("markers", "slow: long-running CPU oracle case")


@pytest.fixture(scope="session")
def fsvd():
    from paper_2605_08314_b200 import build

    build.build()
    import paper_2605_08314_b200 as m

    m.lib()
    return m


@pytest.fixture(scope="session")
def oracle_mod():
    import oracle

    oracle.build(ref=None)
    return oracle


@pytest.fixture(scope="session")
def ref(oracle_mod):
    if not oracle_mod.ref_available():
        pytest.skip("oracle/_ref not built (no /root/reference here); golden fixtures cover this case")
    return oracle_mod.ref()
