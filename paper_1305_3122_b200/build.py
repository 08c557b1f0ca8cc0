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


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _stale():
        return OUT
    cmd = [
        nvcc_path(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-fmad=false",
        "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v",
        "-o", str(OUT) + ".tmp", *[str(CSRC / s) for s in SOURCES],
    ]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        sys.stderr.write(proc.stdout + proc.stderr)
        raise RuntimeError(f"nvcc failed ({proc.returncode})")
    if verbose:
        sys.stderr.write(proc.stderr)
    os.replace(str(OUT) + ".tmp", OUT)
    (PKG_DIR / "build_ptxas.log").write_text(proc.stderr)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
