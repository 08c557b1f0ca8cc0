"""In-tree build of libfemasm_b200.so with nvcc for sm_100a (no JIT, no torch extension).

The library travels to GPU boxes with the repository snapshot, so it is built next to
this file.  ``-fmad=false`` is belt and braces: the value code already uses explicit
round-to-nearest intrinsics, so no FMA contraction can change an element value bit.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
CSRC = PKG_DIR / "csrc"
OUT = PKG_DIR / "libfemasm_b200.so"
SOURCES = ["fa_capi.cu", "fa_assembly.cu", "fa_batch.cu", "fa_triplets.cu", "fa_selftest.cu", "fa_io.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc_path() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not OUT.exists():
        return True
    mtime = OUT.stat().st_mtime
    deps = list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cuh")) + [PKG_DIR.parent / "include" / "femasm_b200.h"]
    return any(p.stat().st_mtime > mtime for p in deps if p.exists())


# checked build (device-side bounds and spin-limit checks, FA_DCHECK in csrc/fa_common.cuh):
# a test artefact loaded by tests/test_checked_build.py, never by the package
OUT_CHECKED = PKG_DIR / "libfemasm_b200_checked.so"


def _stale_for(out: Path) -> bool:
    if not out.exists():
        return True
    mtime = out.stat().st_mtime
    deps = list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cuh")) + [PKG_DIR.parent / "include" / "femasm_b200.h"]
    return any(p.stat().st_mtime > mtime for p in deps if p.exists())


def _nvcc(out: Path, extra: list[str], verbose: bool) -> str:
    cmd = [
        nvcc_path(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-fmad=false",
        "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v", *extra,
        "-o", str(out) + ".tmp", *[str(CSRC / s) for s in SOURCES],
    ]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        sys.stderr.write(proc.stdout + proc.stderr)
        raise RuntimeError(f"nvcc failed ({proc.returncode})")
    if verbose:
        sys.stderr.write(proc.stderr)
    os.replace(str(out) + ".tmp", out)
    return proc.stderr


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _stale():
        return OUT
    (PKG_DIR / "build_ptxas.log").write_text(_nvcc(OUT, [], verbose))
    return OUT


def build_checked(force: bool = False) -> Path:
    if force or _stale_for(OUT_CHECKED):
        _nvcc(OUT_CHECKED, ["-DFA_CHECKED"], False)
    return OUT_CHECKED


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
    if "--checked" in sys.argv:
        print(build_checked(force="--force" in sys.argv))
