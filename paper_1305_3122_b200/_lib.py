"""ctypes binding of the C ABI in include/femasm_b200.h (libfemasm_b200.so).

The shared library is built in-tree by ``paper_1305_3122_b200.build.build()`` (nvcc,
sm_100a).  There is no CPU fallback: if the library or a CUDA device is missing every
compute entry point raises ``RuntimeError``.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

LIB_NAME = "libfemasm_b200.so"
LIB_PATH = Path(os.environ.get("FEMASM_B200_LIB", Path(__file__).resolve().parent / LIB_NAME))

FA_OK = 0
FA_ERR_ARGUMENT = 1
FA_ERR_DEGENERATE = 2
FA_ERR_INDEX = 3
FA_ERR_CUDA = 4
FA_ERR_TOO_LARGE = 5
FA_ERR_LENGTH = 6

KIND_CODES = {"mass": 0, "massw": 1, "stiff": 2, "elastic": 3}

FA_TRIPLETS_KEEP_ZEROS = 1  # CscBuilder semantics (include/femasm_b200.h)

INT64_MAX = np.iinfo(np.int64).max

# Every symbol include/femasm_b200.h declares (checked by tests/test_boundary.py).
EXPORTED_SYMBOLS = (
    "fa_result_status",
    "fa_last_error",
    "fa_version",
    "fa_plan_create",
    "fa_plan_build",
    "fa_plan_capacity",
    "fa_plan_rows",
    "fa_plan_destroy",
    "fa_assemble",
    "fa_assemble_cold",
    "fa_element_kg",
    "fa_build_ig_jg",
    "fa_batch_gradients",
    "fa_compute_areas",
    "fa_mesh_ingest",
    "fa_triplets_workspace",
    "fa_triplets_to_csc",
    "fa_triplets_to_csc_ex",
    "fa_element_triplets",
    "fa_selftest_division",
    "fa_set_kernel_timer",
    "fa_write_matrix_market",
    "fa_read_mesh_text",
)


class FaResult(ctypes.Structure):
    """Mirror of ``fa_result``."""

    _fields_ = [
        ("nnz", ctypes.c_int64),
        ("degenerate_index", ctypes.c_int64),
        ("index_error_pos", ctypes.c_int64),
        ("col_error_pos", ctypes.c_int64),
        ("dropped", ctypes.c_int64),
        ("heavy_rows", ctypes.c_int64),
        ("reserved", ctypes.c_int64 * 1),
        ("repeat_error_pos", ctypes.c_int64),
    ]


RESULT_WORDS = ctypes.sizeof(FaResult) // 8


def result_from_words(words) -> FaResult:
    """An FaResult from the block's RESULT_WORDS int64 words (a host copy of the device block)."""
    r = FaResult()
    off = 0
    for name, typ in FaResult._fields_:
        if not issubclass(typ, ctypes.Array):
            setattr(r, name, int(words[off]))
        off += ctypes.sizeof(typ) // 8
    return r

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_D = ctypes.c_double
_I = ctypes.c_int

_SIGNATURES = {
    "fa_result_status": (_I, [_P]),
    "fa_last_error": (ctypes.c_char_p, []),
    "fa_version": (ctypes.c_char_p, []),
    "fa_plan_create": (_I, [ctypes.POINTER(_P), _I64, _I64, _I64, _I64]),
    "fa_plan_build": (_I, [_P, _P, _P, _P]),
    "fa_plan_capacity": (_I, [_P, _I, ctypes.POINTER(_I64)]),
    "fa_plan_rows": (_I64, [_P, _I]),
    "fa_plan_destroy": (_I, [_P]),
    "fa_assemble": (_I, [_P, _I, _P, _P, _P, _D, _D, _P, _P, _P, _I64, _P, _P]),
    "fa_assemble_cold": (_I, [_P, _P, _I, _P, _P, _P, _D, _D, _P, _P, _P, _I64, _P, _P, _P]),
    "fa_element_kg": (_I, [_I, _P, _I64, _P, _P, _P, _D, _D, _P, _P, _P]),
    "fa_build_ig_jg": (_I, [_I, _P, _I64, _P, _P, _P]),
    "fa_batch_gradients": (_I, [_P, _I64, _P, _P, _P, _P, _P]),
    "fa_compute_areas": (_I, [_P, _I64, _P, _P, _P, _P]),
    "fa_mesh_ingest": (_I, [_P, _I64, _I64, _P, _P, _P, _P, _P]),
    "fa_triplets_workspace": (ctypes.c_size_t, [_I64, _I64, _I64]),
    "fa_triplets_to_csc": (_I, [_P, _P, _P, _I64, _I64, _I64, _P, _P, _P, _P, ctypes.c_size_t, _P, _P]),
    "fa_triplets_to_csc_ex": (_I, [_P, _P, _P, _I64, _I64, _I64, _I, _P, _P, _P, _P, ctypes.c_size_t, _P, _P]),
    "fa_element_triplets": (_I, [_I, _P, _I64, _P, _P, _P, _D, _D, _P, _P, _P, _P, _P]),
    "fa_selftest_division": (_I, [_I64, ctypes.c_uint64, _P, _P, _P]),
    "fa_set_kernel_timer": (_I, [_P, _P]),
    "fa_write_matrix_market": (_I, [ctypes.c_char_p, _I64, _I64, _P, _P, _P, _I]),
    "fa_read_mesh_text": (_I, [ctypes.c_char_p, ctypes.POINTER(_I64), ctypes.POINTER(_I64), _P, _P, _I]),
}

_lib = None


def load_library(path: os.PathLike | str | None = None) -> ctypes.CDLL:
    """Load (once) and type the shared library.  Raises RuntimeError when it is missing."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path is not None else LIB_PATH
    if not p.exists():
        raise RuntimeError(
            f"{p} not found: build the CUDA library first "
            "(python -c 'import paper_1305_3122_b200.build as b; b.build()')"
        )
    lib = ctypes.CDLL(str(p))
    for name, (restype, argtypes) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = restype
        fn.argtypes = argtypes
    if path is None:
        _lib = lib
    return lib


def lib() -> ctypes.CDLL:
    return load_library()


def last_error() -> str:
    msg = lib().fa_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str = "") -> None:
    """Raise the reference's exception type for a failed C-ABI call."""
    if rc == FA_OK:
        return
    msg = last_error() or what
    if rc in (FA_ERR_ARGUMENT, FA_ERR_LENGTH, FA_ERR_INDEX, FA_ERR_DEGENERATE):
        raise ValueError(msg)
    raise RuntimeError(f"femasm_b200 error {rc}: {msg}")


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None for None)."""
    if t is None:
        return None
    return t.data_ptr()


def stream_handle(stream=None) -> int | None:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream or None
