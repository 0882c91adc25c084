"""Compile the NVRTC lanes / segment kernels on the host (no GPU needed).

The lanes and segment kernels are built at run time by NVRTC (csrc/jit.cu,
make_source / seg_source); a compile error there only shows on a GPU box as
"operation not supported" from the launcher.  This restates the two source
builders for a fixed handler list and compiles every template combination the
launchers use with the options of jit.cu's get_compiled, so the CPU suite
catches NVRTC errors.

    python tools/nvrtc_check.py            (prints one line per variant)
"""
from __future__ import annotations

import itertools
import sys
from pathlib import Path

CSRC = Path(__file__).resolve().parents[1] / "paper_2006_03318_b200" / "csrc"
OPTS = [b"--gpu-architecture=sm_100a", b"-std=c++17", b"-lineinfo", b"--device-int128"]
CODES = [0, 1 | (3 << 2), 2 | (1 << 7)]  # a few handler codes (lane / pred-count / flag fields)


def _hstep(c: int) -> str:
    return f"{c & 3}, {(c >> 2) & 31}, {(c >> 7) & 1}"


def lanes_source(dk: int, V: int, dyn: bool, ch: bool, nolb: bool, scale: bool) -> str:
    disp = "#define DDSIM_DISPATCH(h) "
    if dyn:
        disp += "hstep_dyn<V>(S, h, d0, d1, gap, sp, ld, store); if (0) "
    for i, c in enumerate(CODES):
        disp += ("else if (h == " if i else "if (h == ") + \
            f"{c}u) hstep<{_hstep(c)}, V>(S, d0, d1, gap, sp, ld, store); "
    disp += "else __trap();\n"
    src = "#define DDSIM_LANES_NO_STD_TYPES 1\n"
    if dk == 0 and not scale:
        src += "#define DDSIM_DERIVED_SCALE 0\n"
    src += "#define DDSIM_UNROLL 2\n"
    if nolb:
        src += "#define DDSIM_NO_LB 1\n"
    src += disp + (CSRC / "lanes_body.cuh").read_text()
    args = ", const __grid_constant__ ddsim_lanes::ChainParams cp" if ch else ""
    args += ", const __grid_constant__ ddsim_lanes::DerivedParams dp" if dk == 0 else ""
    call = (f"ddsim_lanes::lanes_body<{dk}, {V}, {'true' if ch else 'false'}, false>(&tmap, p, "
            f"{'&cp' if ch else 'nullptr'}, nullptr, 0, 0, nullptr, &dp);" if dk == 0 else
            f"ddsim_lanes::lanes_body<{dk}, {V}, {'true' if ch else 'false'}>(&tmap, p"
            f"{', &cp' if ch else ''});")
    src += ("\nextern \"C\" __global__ void __launch_bounds__(256) ddsim_lanes_jit("
            "const __grid_constant__ ddsim_lanes::Tmap tmap, const ddsim_lanes::Params p"
            f"{args}) {{\n  {call}\n}}\n")
    return src


def seg_source(dk: int, LN: int, ch: bool, mode: int, scale: bool) -> str:
    src = "#define DDSIM_LANES_NO_STD_TYPES 1\n"
    if dk == 0 and not scale:
        src += "#define DDSIM_DERIVED_SCALE 0\n"
    if dk != 0:
        src += "#define DDSIM_UNROLL 2\n#define DDSIM_STAGES 2\n"
    disp = "#define DDSIM_DISPATCH(h) "
    sdisp = "#define DDSIM_SYM_DISPATCH(h) "
    sdisp2 = "#define DDSIM_SYM_DISPATCH2(h) "
    for i, c in enumerate(CODES):
        cond = ("else if (h == " if i else "if (h == ") + f"{c}u) "
        disp += cond + f"hstep<{_hstep(c)}, V>(S, d0, d1, gap, sp, ld, store); "
        sdisp += cond + f"hsym<{_hstep(c)}, LN>(Y, dv, gp); "
        sdisp2 += cond + f"{{ hsym<{_hstep(c)}, LN>(Y, dv, gp); hsym<{_hstep(c)}, LN>(Y2, dv2, gp); }} "
    src += disp + "else __trap();\n" + sdisp + "else __trap();\n" + sdisp2 + "else __trap();\n"
    src += (CSRC / "lanes_body.cuh").read_text() + "\n" + (CSRC / "lanes_seg.cuh").read_text() + "\n"
    name = ["ddsim_seg_replay", "ddsim_seg_transfer", "ddsim_seg_fused", "ddsim_seg_transfer2",
            "ddsim_seg_replay2"][mode]
    body = ["replay_body", "sym_body", "fused_body", "sym_body2", "replay_body2"][mode]
    args = ", const __grid_constant__ ddsim_lanes::ChainParams cp" if ch else ""
    args += ", const __grid_constant__ ddsim_lanes::DerivedParams dp" if dk == 0 else ""
    return src + (f"extern \"C\" __global__ void __launch_bounds__(256) {name}("
                  "const __grid_constant__ ddsim_lanes::Tmap tmap, const ddsim_lanes::Params p, "
                  f"const ddsim_lanes::SegParams sg{args}) {{\n  ddsim_lanes::{body}<{dk}, {LN}, "
                  f"{'true' if ch else 'false'}>(&tmap, p, sg, {'&cp' if ch else 'nullptr'}"
                  f"{', &dp' if dk == 0 else ', nullptr'});\n}}\n")


def compile_source(src: str) -> tuple[bool, str]:
    from cuda.bindings import nvrtc
    err, prog = nvrtc.nvrtcCreateProgram(src.encode(), b"ddsim_lanes_jit.cu", 0, [], [])
    assert err == nvrtc.nvrtcResult.NVRTC_SUCCESS
    try:
        (rc,) = nvrtc.nvrtcCompileProgram(prog, len(OPTS), OPTS)
        err, n = nvrtc.nvrtcGetProgramLogSize(prog)
        log = b" " * n
        nvrtc.nvrtcGetProgramLog(prog, log)
        return rc == nvrtc.nvrtcResult.NVRTC_SUCCESS, log.decode(errors="replace").strip("\x00 \n")
    finally:
        nvrtc.nvrtcDestroyProgram(prog)


def variants():
    """The combinations the launchers request (maxplus_lanes.cu / jit.cu)."""
    for dk, V, ch in itertools.product((0, 1, 2), (1, 2), (False, True)):
        if dk == 0 and V != 1:
            continue  # derived durations: one scenario per thread
        for dyn, nolb in ((False, False), (True, False), (False, True)):
            yield f"lanes dk={dk} V={V} ch={ch} dyn={dyn} nolb={nolb}", \
                lanes_source(dk, V, dyn, ch, nolb, scale=True)
        if dk == 0:
            yield f"lanes dk=0 V=1 ch={ch} noscale", lanes_source(0, 1, False, ch, False, False)
    for dk, LN, ch, mode in itertools.product((0, 1, 2), (2, 3), (False, True), (0, 1, 3, 4)):
        yield f"seg dk={dk} LN={LN} ch={ch} mode={mode}", seg_source(dk, LN, ch, mode, True)
    for dk in (1, 2):
        yield f"seg dk={dk} LN=4 mode=3", seg_source(dk, 4, False, 3, True)
    for mode in (0, 3, 4):
        yield f"seg dk=0 LN=3 ch=True mode={mode} noscale", seg_source(0, 3, True, mode, False)


def main(argv=None) -> int:
    bad = 0
    for name, src in variants():
        ok, log = compile_source(src)
        print(("ok   " if ok else "FAIL ") + name, flush=True)
        if not ok:
            bad += 1
            print(log[:4000])
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))
