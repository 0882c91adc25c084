"""The NVRTC-built lanes / segment kernels compile for sm_100a (host NVRTC, no
GPU): every template combination the launchers request (tools/nvrtc_check.py
restates jit.cu's make_source / seg_source)."""
import sys
from pathlib import Path

import pytest

sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tools"))
nvrtc = pytest.importorskip("cuda.bindings.nvrtc")
import nvrtc_check  # noqa: E402

VARIANTS = list(nvrtc_check.variants())


@pytest.mark.parametrize("name,src", VARIANTS, ids=[v[0] for v in VARIANTS])
def test_jit_source_compiles(name, src):
    ok, log = nvrtc_check.compile_source(src)
    assert ok, log[:4000]
