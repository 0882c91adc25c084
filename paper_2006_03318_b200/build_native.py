"""Build libddsim.so (sm_100a) and the oracle library with plain nvcc/gcc.

Run: ``python -m paper_2006_03318_b200.build_native`` (or __graft_entry__.build()).
Objects are compiled in parallel and linked into an in-tree shared object so
it travels to the GPU box with the repository snapshot.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = ROOT / "build" / "native"
LIB = PKG / "libddsim.so"
ORACLE_SRC = ROOT / "oracle" / "ddsim_oracle.c"
ORACLE_LIB = ROOT / "oracle" / "liboracle.so"

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2",
    "--expt-relaxed-constexpr", "-Xptxas", "-v",
]


GXX_FLAGS = ["-O3", "-std=c++17", "-fPIC", "-pthread", "-Wall", "-Wno-unused-function"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _run(cmd: list[str], log: Path | None = None) -> str:
    p = subprocess.run(cmd, capture_output=True, text=True)
    out = p.stdout + p.stderr
    if log is not None:
        log.write_text(out)
    if p.returncode != 0:
        raise RuntimeError(f"command failed: {' '.join(cmd)}\n{out}")
    return out


def _embed_sources() -> None:
    """NVRTC source texts: csrc/lanes_body.cuh -> generated/lanes_body_src.inc,
    csrc/lanes_seg.cuh -> generated/lanes_seg_src.inc (generated at build time,
    not tracked)."""
    gen = CSRC / "generated"
    gen.mkdir(exist_ok=True)
    for src, name, var in (("lanes_body.cuh", "lanes_body_src.inc", "kLanesBodySrc"),
                           ("lanes_seg.cuh", "lanes_seg_src.inc", "kSegBodySrc")):
        body = (CSRC / src).read_text()
        out = gen / name
        text = f'static const char* {var} = R"DDSIM_SRC(' + body + ')DDSIM_SRC";\n'
        if not out.exists() or out.read_text() != text:
            out.write_text(text)


def build_library(verbose: bool = False) -> Path:
    BUILD.mkdir(parents=True, exist_ok=True)
    _embed_sources()
    nvcc = _nvcc()
    sources = sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cpp"))
    headers = (sorted(CSRC.glob("*.h")) + sorted(CSRC.glob("*.cuh"))
               + sorted((CSRC / "generated").glob("*.inc")) + [ROOT / "include" / "ddsim.h"])
    newest_h = max(h.stat().st_mtime for h in headers)

    def compile_one(src: Path) -> Path:
        obj = BUILD / (src.stem + ".o")
        if obj.exists() and obj.stat().st_mtime > max(src.stat().st_mtime, newest_h):
            return obj
        if src.suffix == ".cpp":  # host-only code: plain g++
            _run(["g++", *GXX_FLAGS, "-I", str(ROOT / "include"), "-c", str(src), "-o", str(obj)],
                 BUILD / (src.stem + ".gxx.log"))
        else:
            _run([nvcc, *NVCC_FLAGS, "-I", str(ROOT / "include"), "-c", str(src), "-o", str(obj)],
                 BUILD / (src.stem + ".ptxas.log"))
        return obj

    with ThreadPoolExecutor(max_workers=min(8, len(sources))) as ex:
        objs = list(ex.map(compile_one, sources))
    tmp = LIB.with_suffix(".so.tmp")
    _run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(tmp),
          *map(str, objs), "-lcudart_static", "-lrt", "-ldl", "-lpthread"])
    os.replace(tmp, LIB)
    if verbose:
        print(f"built {LIB}")
    return LIB


def build_oracle(verbose: bool = False) -> Path:
    if ORACLE_LIB.exists() and ORACLE_LIB.stat().st_mtime > ORACLE_SRC.stat().st_mtime:
        return ORACLE_LIB
    _run(["gcc", "-O2", "-fPIC", "-shared", "-o", str(ORACLE_LIB), str(ORACLE_SRC), "-lpthread"])
    if verbose:
        print(f"built {ORACLE_LIB}")
    return ORACLE_LIB


def main() -> int:
    build_library(verbose=True)
    build_oracle(verbose=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
