import gzip
import json
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
for p in (ROOT, ROOT / "oracle", ROOT / "tests"):
    if str(p) not in sys.path:
        sys.path.insert(0, str(p))

GOLDEN = ROOT / "tests" / "golden" / "golden.json.gz"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


@pytest.fixture(scope="session")
def golden():
    with gzip.open(GOLDEN, "rt") as fh:
        return json.load(fh)


def has_gpu() -> bool:
    try:
        from paper_2006_03318_b200 import _native
        return _native.device_count() > 0
    except Exception:  # noqa: BLE001
        return False
