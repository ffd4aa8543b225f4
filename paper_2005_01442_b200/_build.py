"""Build recipe for the sm_100a extension (called by __graft_entry__.build()).

Compiles every csrc/*.cu into one shared library, in-tree, so it travels to the
GPU box with the repo snapshot:

    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false ...

-fmad=false keeps every float64 multiply and add separately rounded (the
parity mode, SURVEY 7 hard part (i)); explicit fma() calls are unaffected.
"""

from __future__ import annotations

import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
ROOT = PKG.parent
LIB_NAME = "libvoxelray_b200.so"
LIB_PATH = PKG / LIB_NAME

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    "-O3", "-lineinfo", "-std=c++17", "-fmad=false", "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC,-O2", "-Xptxas", "-v", "-shared", "-cudart", "static",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; the CUDA toolkit is required to build the extension")


def sources():
    return sorted(CSRC.glob("*.cu"))


def deps():
    return sources() + sorted(CSRC.glob("*.cuh")) + [ROOT / "include" / "voxelray_b200.h", Path(__file__)]


def up_to_date() -> bool:
    if not LIB_PATH.exists():
        return False
    t = LIB_PATH.stat().st_mtime
    return all(p.stat().st_mtime <= t for p in deps())


def build(force: bool = False, verbose: bool = False, out: Path | None = None,
          defines: tuple[str, ...] = ()) -> Path:
    """Compile the library (to ``out`` with extra -D ``defines`` for experiments)."""
    target = Path(out) if out else LIB_PATH
    if not force and out is None and not defines and up_to_date():
        return LIB_PATH
    tmp = target.with_suffix(".so.tmp")
    cmd = [nvcc(), *ARCH, *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-I", str(ROOT / "include"),
           *map(str, sources()), "-o", str(tmp)]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    log = target.with_suffix(".build.log") if out else PKG / "build.log"
    log.write_text(" ".join(cmd) + "\n" + proc.stdout + proc.stderr)
    if proc.returncode != 0:
        raise RuntimeError(f"nvcc failed ({proc.returncode}); see {log}\n{proc.stderr[-4000:]}")
    os.replace(tmp, target)
    if verbose:
        print(proc.stderr)
    return target


if __name__ == "__main__":
    import sys

    if len(sys.argv) > 2:  # _build.py OUT.so DEFINE [DEFINE ...]
        print(build(force=True, out=Path(sys.argv[1]), defines=tuple(sys.argv[2:])))
    else:
        print(build(force=True, verbose=True))
