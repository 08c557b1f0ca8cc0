"""ctypes wrapper of oracle/c/femasm_oracle.c — TEST INFRASTRUCTURE ONLY.

Fast CPU restatement of the reference OptV2 assembly (see the C file header) used for
parity checks at BASELINE sizes and pinned against the numpy oracle and the reference
digests (tests/test_oracle_golden.py).
"""

from __future__ import annotations

import ctypes
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "build" / "libfemasm_oracle.so"
KIND = {"mass": 0, "massw": 1, "stiff": 2, "elastic": 3}

_lib = None


def build(force: bool = False) -> Path:
    src = HERE / "c" / "femasm_oracle.c"
    if force or not LIB.exists() or LIB.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(str(LIB))
        P, I64, D, I = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_int
        L.fo_capacity.restype = I64
        L.fo_capacity.argtypes = [I, I64, P, I64, I64]
        L.fo_assemble.restype = I64
        L.fo_assemble.argtypes = [I, I64, P, P, P, P, D, D, I64, I64, P, P, P, ctypes.POINTER(I64)]
        L.fo_areas.restype = None
        L.fo_areas.argtypes = [I64, P, P, P]
        L.fo_element_values.restype = None
        L.fo_element_values.argtypes = [I, I64, P, P, P, P, D, D, P]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data


def areas(q, me):
    q = np.ascontiguousarray(q, dtype=np.float64)
    me = np.ascontiguousarray(me, dtype=np.int64)
    out = np.empty(me.shape[0])
    lib().fo_areas(me.shape[0], _p(q), _p(me), _p(out))
    return out


def element_values(kind, q, me, areas_, w=None, lam=0.0, mu=0.0):
    me = np.ascontiguousarray(me, dtype=np.int64)
    q = None if q is None else np.ascontiguousarray(q, dtype=np.float64)
    areas_ = np.ascontiguousarray(areas_, dtype=np.float64)
    w = None if w is None else np.ascontiguousarray(w, dtype=np.float64)
    r = 36 if kind == "elastic" else 9
    kg = np.empty((r, me.shape[0]))
    lib().fo_element_values(KIND[kind], me.shape[0], _p(q), _p(me), _p(areas_), _p(w), float(lam), float(mu), _p(kg))
    return kg


def assemble(kind, q, me, areas_, w=None, lam=0.0, mu=0.0, col_begin=0, col_end=None):
    """CSC arrays (colptr local to the column block, rowidx, vals) of columns
    [col_begin, col_end) (dof numbering; default: all)."""
    me = np.ascontiguousarray(me, dtype=np.int64)
    q = None if q is None else np.ascontiguousarray(q, dtype=np.float64)
    areas_ = np.ascontiguousarray(areas_, dtype=np.float64)
    w = None if w is None else np.ascontiguousarray(w, dtype=np.float64)
    nq = q.shape[0] if q is not None else (w.shape[0] if w is not None else int(me.max()) + 1)
    n = 2 * nq if kind == "elastic" else nq
    col_end = n if col_end is None else int(col_end)
    L = lib()
    cap = L.fo_capacity(KIND[kind], me.shape[0], _p(me), int(col_begin), col_end)
    colptr = np.empty(col_end - col_begin + 1, dtype=np.int64)
    rowidx = np.empty(max(cap, 1), dtype=np.int64)
    vals = np.empty(max(cap, 1))
    bad = ctypes.c_int64(-1)
    nnz = L.fo_assemble(KIND[kind], me.shape[0], _p(q), _p(me), _p(areas_), _p(w), float(lam), float(mu),
                        int(col_begin), col_end, _p(colptr), _p(rowidx), _p(vals), ctypes.byref(bad))
    if nnz < 0:
        raise MemoryError("oracle allocation failed")
    if bad.value >= 0:
        raise ValueError(f"triangle {bad.value} is degenerate")
    return colptr, rowidx[:nnz].copy(), vals[:nnz].copy()
