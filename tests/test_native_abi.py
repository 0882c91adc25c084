"""The C-ABI library loads and exports every symbol include/ddsim.h declares
(no compute calls here: CPU only)."""

import re
from pathlib import Path

import pytest

from paper_2006_03318_b200 import _native as N

HEADER = Path(__file__).resolve().parents[1] / "include" / "ddsim.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(ks_[a-z_]+)\s*\(", text)))


def test_header_declares_what_the_binding_binds():
    assert declared_symbols() == sorted(N.EXPORTED_SYMBOLS)


def test_library_exports_every_declared_symbol():
    lib = N.lib()
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_error_names_match_reference_taxonomy():
    lib = N.lib()
    names = {code: lib.ks_error_name(code).decode() for code in range(0, 12)}
    assert names[N.KS_ERR_DEADLOCK] == "Deadlock"
    assert names[N.KS_ERR_CYCLE] == "CycleDetected"
    assert names[N.KS_ERR_ORPHAN] == "OrphanKernel"
    assert names[N.KS_ERR_AMBIGUOUS] == "AmbiguousMarker"
    assert names[N.KS_ERR_OVERLAP] == "OverlapViolation"
    assert names[N.KS_ERR_BAD_PIPELINE] == "BadPipeline"
    from paper_2006_03318_b200 import errors
    for code, name in names.items():
        if code and name not in ("InvalidArgument",):
            assert hasattr(errors, name), name


def test_struct_layouts_match_header():
    import ctypes as C
    assert C.sizeof(N.ScaleStep) == 24
    assert N.SCALE_STEP_DTYPE.itemsize == 24
    assert C.sizeof(N.SimOut) == 48
    # 2 ints + 8 pointers + int64 + 4 pointers + int32(+pad) + 4 pointers
    assert C.sizeof(N.GraphDesc) == 8 + 8 * 8 + 8 + 4 * 8 + 8 + 4 * 8


def test_no_cpu_fallback_without_device():
    """Without a GPU every compute entry point must raise, not fall back."""
    if N.device_count() > 0:
        pytest.skip("a device is present")
    from paper_2006_03318_b200 import errors, simulate
    from paper_2006_03318_b200.graph import DependencyGraph, Task
    from paper_2006_03318_b200.trace import LaneId, TaskKind
    g = DependencyGraph()
    g.tasks[0] = Task(id=0, kind=TaskKind.CPU_OTHER, name="a", lane=LaneId.parse("cpu:0"),
                      duration=5)
    g.lane_order[LaneId.parse("cpu:0")] = [0]
    with pytest.raises(errors.NoDevice):
        simulate(g)
