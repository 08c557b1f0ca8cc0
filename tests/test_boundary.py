"""The C-ABI boundary: the library loads (no GPU needed) and exports exactly what
include/femasm_b200.h declares; argument errors map to the reference's exception types."""

import ctypes
import re
from pathlib import Path

import pytest

from paper_1305_3122_b200 import _lib

HEADER = Path(__file__).resolve().parents[1] / "include" / "femasm_b200.h"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fa_[a-z_0-9]+)\s*\(", text)))


def test_library_loads_and_exports_every_declared_symbol():
    lib = _lib.load_library()
    names = declared_functions()
    assert names, "no declarations parsed"
    for name in names:
        assert hasattr(lib, name), f"{name} declared in femasm_b200.h but not exported"
    assert sorted(_lib.EXPORTED_SYMBOLS) == names


def test_version_and_result_status_without_gpu():
    lib = _lib.load_library()
    assert b"sm_100a" in lib.fa_version()
    r = _lib.FaResult()
    r.index_error_pos = _lib.INT64_MAX
    r.col_error_pos = _lib.INT64_MAX
    r.degenerate_index = _lib.INT64_MAX
    r.repeat_error_pos = _lib.INT64_MAX
    assert lib.fa_result_status(ctypes.addressof(r)) == _lib.FA_OK
    r.repeat_error_pos = 5
    assert lib.fa_result_status(ctypes.addressof(r)) == _lib.FA_ERR_INDEX
    r.repeat_error_pos = _lib.INT64_MAX
    r.degenerate_index = 3
    assert lib.fa_result_status(ctypes.addressof(r)) == _lib.FA_ERR_DEGENERATE
    r.index_error_pos = 0
    assert lib.fa_result_status(ctypes.addressof(r)) == _lib.FA_ERR_INDEX
    assert ctypes.sizeof(_lib.FaResult) == 64


def test_result_words_map_to_fields():
    words = list(range(10, 10 + _lib.RESULT_WORDS))
    r = _lib.result_from_words(words)
    assert (r.nnz, r.degenerate_index, r.index_error_pos, r.col_error_pos) == (10, 11, 12, 13)
    assert (r.dropped, r.heavy_rows, r.repeat_error_pos) == (14, 15, 17)


def test_plan_argument_errors_are_reported_before_touching_the_device():
    lib = _lib.load_library()
    h = ctypes.c_void_p()
    assert lib.fa_plan_create(ctypes.byref(h), 0, 3, 0, 3) == _lib.FA_ERR_ARGUMENT
    assert "at least one" in _lib.last_error()
    assert lib.fa_plan_create(ctypes.byref(h), 4, 3, 2, 5) == _lib.FA_ERR_ARGUMENT
    assert "row block" in _lib.last_error()
    assert lib.fa_plan_create(ctypes.byref(h), 2**31, 3, 0, 3) == _lib.FA_ERR_TOO_LARGE
    assert lib.fa_plan_create(None, 1, 3, 0, 3) == _lib.FA_ERR_ARGUMENT
    with pytest.raises(ValueError):
        _lib.check(_lib.FA_ERR_ARGUMENT)
    with pytest.raises(RuntimeError):
        _lib.check(_lib.FA_ERR_CUDA)


def test_kernel_entry_points_validate_arguments():
    lib = _lib.load_library()
    assert lib.fa_element_kg(7, None, 1, None, None, None, 0.0, 0.0, None, None, None) == _lib.FA_ERR_ARGUMENT
    assert "unknown matrix kind" in _lib.last_error()
    assert lib.fa_assemble(None, 0, None, None, None, 0.0, 0.0, None, None, None, 0, None, None) == _lib.FA_ERR_ARGUMENT
    assert lib.fa_assemble_cold(None, None, 0, None, None, None, 0.0, 0.0, None, None, None, 0, None, None,
                                None) == _lib.FA_ERR_ARGUMENT
    assert lib.fa_triplets_to_csc(None, None, None, 0, 0, 3, None, None, None, None, 0, None, None) == _lib.FA_ERR_ARGUMENT
    assert lib.fa_triplets_workspace(1000, 10, 10) > 1000 * 32


def test_header_cites_the_reference_interfaces():
    text = HEADER.read_text()
    for cite in ("assembly.py:214", "assembly.py:162-192", "sparse.py:140-189", "mesh.py:51-69"):
        assert cite in text
