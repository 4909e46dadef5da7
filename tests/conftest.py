import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through libscmwu.so)")
    config.addinivalue_line("markers", "slow: long CPU test")


def load_golden(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


def gf(x):
    """Decode a golden float (inf encoded as a string)."""
    if isinstance(x, str):
        return float(x)
    return x


@pytest.fixture(scope="session")
def golden():
    return {n: load_golden(n + ".json") for n in ("kats", "traces", "calls", "long",
                                                    "generators")}


@pytest.fixture(scope="session")
def emu_engine():
    """CPU emulation of the engine (tests only; never used by the package)."""
    import build
    from paper_2405_09157_b200 import _native as nat
    return nat.Engine(build.build_emu())


@pytest.fixture(scope="session")
def cuda_engine():
    from paper_2405_09157_b200 import _native as nat
    return nat.cuda_engine()
