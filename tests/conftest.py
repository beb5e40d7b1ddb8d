import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) device; parity tests through the C ABI")


def _ensure_built():
    from paper_2203_10000_b200 import _native, build
    oracle_libs = [ROOT / "oracle" / "build" / f for f in ("liblabel_oracle.so", "librefine_oracle.so")]
    if not (_native.LABEL_LIB.exists() and _native.SYNTH_LIB.exists() and all(p.exists() for p in oracle_libs)):
        build.build_all()


_ensure_built()


@pytest.fixture(scope="session")
def has_gpu():
    from paper_2203_10000_b200._native import cuda_device_available
    return cuda_device_available()


@pytest.fixture(scope="session")
def ctx():
    """One labeling context on cuda:0 for the whole GPU session."""
    from paper_2203_10000_b200._native import Context
    c = Context(0)
    yield c
    c.close()
