"""Compressed sparse matrices (mirror of femasm.sparse, /root/reference/pkg/src/femasm/sparse.py).

``csc_from_triplets`` keeps Matlab ``sparse`` semantics (input zeros ignored, duplicates
summed left to right in input order, exact-zero sums dropped, sparse.py:140-189) but runs
on the GPU (fa_triplets_to_csc: stable LSD radix sort of (code, value) pairs with shared-memory-staged tiles + sequential run sums).
``CscMatrix`` has the reference's immutable host interface (col_ptr/row_idx int64, values
f64) and can also wrap a device CSR produced by ``assemble``; its host arrays are then
materialised on first access.  ``CscBuilder`` — the deliberately quadratic insertion
builder of the reference's complexity study (sparse.py:208-291) — is out of scope for the
B200 path and kept as a thin host-side container so element-loop callers still work.
"""

from __future__ import annotations

from dataclasses import dataclass

import os

import numpy as np

from . import _lib
from .device import ResultBlock, device, require_cuda

__all__ = [
    "CscBuilder",
    "CscMatrix",
    "TripletBatch",
    "csc_from_triplets",
    "max_abs_diff",
    "write_matrix_market",
]

DENSE_LIMIT = 10**8  # sparse.py:36


class CscMatrix:
    """Immutable CSC matrix (sparse.py:39-121).  For assembled (symmetric) matrices the
    device CSR arrays are these CSC arrays bit for bit."""

    __slots__ = ("n_rows", "n_cols", "_col_ptr", "_row_idx", "_values", "_dev")

    def __init__(self, n_rows, n_cols, col_ptr, row_idx, values, validate=True):
        n_rows, n_cols = int(n_rows), int(n_cols)
        if n_rows < 1 or n_cols < 1:
            raise ValueError("matrix dimensions must be positive")
        col_ptr = np.ascontiguousarray(col_ptr, dtype=np.int64)
        row_idx = np.ascontiguousarray(row_idx, dtype=np.int64)
        values = np.ascontiguousarray(values, dtype=np.float64)
        if validate:
            _validate_csc(n_rows, n_cols, col_ptr, row_idx, values)
        for arr in (col_ptr, row_idx, values):
            arr.flags.writeable = False
        object.__setattr__(self, "n_rows", n_rows)
        object.__setattr__(self, "n_cols", n_cols)
        object.__setattr__(self, "_col_ptr", col_ptr)
        object.__setattr__(self, "_row_idx", row_idx)
        object.__setattr__(self, "_values", values)
        object.__setattr__(self, "_dev", None)

    @classmethod
    def from_device(cls, n_rows, n_cols, ptr, idx, vals) -> "CscMatrix":
        """Wrap device arrays (ptr int64, idx int32/int64, vals f64) without copying."""
        m = cls.__new__(cls)
        object.__setattr__(m, "n_rows", int(n_rows))
        object.__setattr__(m, "n_cols", int(n_cols))
        object.__setattr__(m, "_col_ptr", None)
        object.__setattr__(m, "_row_idx", None)
        object.__setattr__(m, "_values", None)
        object.__setattr__(m, "_dev", (ptr, idx, vals))
        return m

    def _materialise(self) -> None:
        ptr, idx, vals = self._dev
        col_ptr = ptr.cpu().numpy().astype(np.int64, copy=False)
        row_idx = idx.cpu().numpy().astype(np.int64)
        values = vals.cpu().numpy()
        for arr in (col_ptr, row_idx, values):
            arr.flags.writeable = False
        object.__setattr__(self, "_col_ptr", col_ptr)
        object.__setattr__(self, "_row_idx", row_idx)
        object.__setattr__(self, "_values", values)

    @property
    def col_ptr(self) -> np.ndarray:
        if self._col_ptr is None:
            self._materialise()
        return self._col_ptr

    @property
    def row_idx(self) -> np.ndarray:
        if self._row_idx is None:
            self._materialise()
        return self._row_idx

    @property
    def values(self) -> np.ndarray:
        if self._values is None:
            self._materialise()
        return self._values

    def __setattr__(self, name, value):
        raise AttributeError("CscMatrix is immutable")

    @property
    def nnz(self) -> int:
        if self._dev is not None:
            return int(self._dev[2].numel())
        return int(self._values.size)

    @property
    def shape(self) -> tuple[int, int]:
        return (self.n_rows, self.n_cols)

    def device_arrays(self):
        """(ptr int64, idx, vals f64) on the GPU (uploads host-built matrices)."""
        if self._dev is None:
            torch = require_cuda()
            dev = device()
            object.__setattr__(self, "_dev", (
                torch.from_numpy(self._col_ptr.copy()).to(dev),
                torch.from_numpy(self._row_idx.copy()).to(dev),
                torch.from_numpy(self._values.copy()).to(dev),
            ))
        return self._dev

    def get(self, i: int, j: int) -> float:
        """Stored value at (i, j), or 0.0 when the position is absent."""
        if not (0 <= i < self.n_rows and 0 <= j < self.n_cols):
            raise ValueError(f"index ({i}, {j}) out of range for {self.shape}")
        lo, hi = int(self.col_ptr[j]), int(self.col_ptr[j + 1])
        pos = lo + int(np.searchsorted(self.row_idx[lo:hi], i))
        if pos < hi and self.row_idx[pos] == i:
            return float(self.values[pos])
        return 0.0

    def triplets(self):
        """(rows, cols, values) in column-major storage order."""
        cols = np.repeat(np.arange(self.n_cols, dtype=np.int64), np.diff(self.col_ptr))
        return self.row_idx.copy(), cols, self.values.copy()

    def to_dense(self) -> np.ndarray:
        if self.n_rows * self.n_cols > DENSE_LIMIT:
            raise ValueError(f"dense expansion of {self.shape} exceeds the {DENSE_LIMIT} entry guard")
        dense = np.zeros((self.n_rows, self.n_cols))
        rows, cols, vals = self.triplets()
        dense[rows, cols] = vals
        return dense

    def drop_zeros(self) -> "CscMatrix":
        rows, cols, vals = self.triplets()
        return csc_from_triplets(rows, cols, vals, self.n_rows, self.n_cols)

    def to_scipy(self):
        """scipy.sparse.csc_matrix view of the host arrays."""
        import scipy.sparse as sp

        return sp.csc_matrix((self.values, self.row_idx, self.col_ptr), shape=self.shape)

    def to_torch_sparse_csr(self):
        """torch sparse CSR on the device.  Valid as CSR for the symmetric assembled
        matrices (CSC of A == CSR of A^T == CSR of A)."""
        import torch

        ptr, idx, vals = self.device_arrays()
        # torch wants one index dtype: the int32 column ids are handed over as they are (zero
        # copy) and the row pointers narrowed (n+1 entries instead of nnz) whenever nnz fits
        if idx.dtype == torch.int32 and int(self.nnz) < 2**31:
            return torch.sparse_csr_tensor(ptr.to(torch.int32), idx, vals, size=(self.n_cols, self.n_rows))
        return torch.sparse_csr_tensor(ptr, idx.to(torch.int64), vals, size=(self.n_cols, self.n_rows))

    def __repr__(self) -> str:
        return f"CscMatrix(shape={self.shape}, nnz={self.nnz})"


def _validate_csc(n_rows, n_cols, col_ptr, row_idx, values) -> None:
    # same checks and messages as sparse.py:54-70
    if col_ptr.shape != (n_cols + 1,):
        raise ValueError("col_ptr must have n_cols+1 entries")
    if col_ptr[0] != 0 or col_ptr[-1] != row_idx.size:
        raise ValueError("col_ptr must start at 0 and end at nnz")
    if (np.diff(col_ptr) < 0).any():
        raise ValueError("col_ptr must be nondecreasing")
    if row_idx.shape != values.shape:
        raise ValueError("row_idx and values must have equal length")
    if row_idx.size:
        if row_idx.min() < 0 or row_idx.max() >= n_rows:
            raise ValueError("row index out of range")
        starts = np.repeat(np.arange(n_cols), np.diff(col_ptr))
        same_col = starts[1:] == starts[:-1]
        if (np.diff(row_idx)[same_col] <= 0).any():
            raise ValueError("row indices must increase within a column")


def _as_index_array(idx) -> np.ndarray:
    idx = np.asarray(idx)
    if idx.dtype.kind != "i":
        idx = idx.astype(np.int64)
    return np.ascontiguousarray(idx, dtype=np.int64).ravel()


def csc_from_triplets(rows, cols, vals, n_rows: int, n_cols: int) -> CscMatrix:
    """Matlab ``sparse(I, J, K, m, n)`` on the GPU (sparse.py:140-189)."""
    rows = _as_index_array(rows)
    cols = _as_index_array(cols)
    vals = np.ascontiguousarray(vals, dtype=np.float64).ravel()
    if not (rows.size == cols.size == vals.size):
        raise ValueError(f"triplet arrays disagree in length: {rows.size}, {cols.size}, {vals.size}")
    if n_rows < 1 or n_cols < 1:
        raise ValueError("matrix dimensions must be positive")
    torch = require_cuda()
    dev = device()
    d_rows = torch.from_numpy(rows).to(dev)
    d_cols = torch.from_numpy(cols).to(dev)
    d_vals = torch.from_numpy(vals).to(dev)
    return _triplets_device(d_rows, d_cols, d_vals, int(n_rows), int(n_cols), host_rows=rows, host_cols=cols)


def _triplets_device(d_rows, d_cols, d_vals, n_rows, n_cols, host_rows=None, host_cols=None,
                     keep_zeros: bool = False) -> CscMatrix:
    """Device triplets -> CscMatrix: Matlab sparse() (sparse.py:140-189), or with `keep_zeros`
    the CscBuilder semantics of the element-loop strategies (sparse.py:208-290)."""
    torch = require_cuda()
    dev = device()
    n = int(d_vals.numel())
    L = _lib.lib()
    ws_bytes = int(L.fa_triplets_workspace(n, n_rows, n_cols))
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    colptr = torch.empty(n_cols + 1, dtype=torch.int64, device=dev)
    rowidx = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    vout = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
    res = ResultBlock()
    rc = L.fa_triplets_to_csc_ex(
        _lib.ptr(d_rows) if n else None, _lib.ptr(d_cols) if n else None, _lib.ptr(d_vals) if n else None,
        n, n_rows, n_cols, _lib.FA_TRIPLETS_KEEP_ZEROS if keep_zeros else 0, colptr.data_ptr(), rowidx.data_ptr(),
        vout.data_ptr(), ws.data_ptr(), ws_bytes, res.ptr, _lib.stream_handle(),
    )
    _lib.check(rc, "fa_triplets_to_csc")
    r = res.fetch()
    if r.index_error_pos != _lib.INT64_MAX:
        pos = r.index_error_pos
        bad = int(host_rows[pos]) if host_rows is not None else int(d_rows[pos].item())
        raise ValueError(f"row index {bad} at position {pos} out of range [0, {n_rows})")
    if r.col_error_pos != _lib.INT64_MAX:
        pos = r.col_error_pos
        bad = int(host_cols[pos]) if host_cols is not None else int(d_cols[pos].item())
        raise ValueError(f"column index {bad} at position {pos} out of range [0, {n_cols})")
    return CscMatrix.from_device(n_rows, n_cols, colptr, rowidx[: r.nnz], vout[: r.nnz])


def max_abs_diff(a: CscMatrix, b: CscMatrix) -> float:
    """max |a - b| over every position, absent entries counting as zero (sparse.py:192-205)."""
    if a.shape != b.shape:
        raise ValueError(f"shape mismatch: {a.shape} vs {b.shape}")
    ra, ca, va = a.triplets()
    rb, cb, vb = b.triplets()
    diff = csc_from_triplets(np.concatenate([ra, rb]), np.concatenate([ca, cb]), np.concatenate([va, -vb]),
                             a.n_rows, a.n_cols)
    return float(np.abs(diff.values).max()) if diff.nnz else 0.0


class CscBuilder:
    """Incremental CSC image (sparse.py:208-291).  The reference keeps this naive O(nnz)
    insertion on purpose for its complexity study; that study is out of the B200 scope,
    so this mirror keeps a per-column dict and snapshots to CscMatrix (explicit zeros
    kept, like the reference's to_matrix)."""

    __slots__ = ("n_rows", "n_cols", "_cols")

    def __init__(self, n_rows: int, n_cols: int):
        if n_rows < 1 or n_cols < 1:
            raise ValueError("matrix dimensions must be positive")
        self.n_rows = int(n_rows)
        self.n_cols = int(n_cols)
        self._cols = [dict() for _ in range(self.n_cols)]

    @property
    def nnz(self) -> int:
        return sum(len(c) for c in self._cols)

    def add(self, i: int, j: int, v: float) -> None:
        if not (0 <= i < self.n_rows and 0 <= j < self.n_cols):
            raise ValueError(f"index ({i}, {j}) out of range for ({self.n_rows}, {self.n_cols})")
        col = self._cols[j]
        col[i] = col.get(i, 0.0) + v if i in col else float(v)

    def add_block(self, row_ids, col_ids, block) -> None:
        block = np.asarray(block, dtype=np.float64)
        if block.shape != (len(row_ids), len(col_ids)):
            raise ValueError(f"block shape {block.shape} does not match ids ({len(row_ids)}, {len(col_ids)})")
        for b, j in enumerate(col_ids):
            for a, i in enumerate(row_ids):
                self.add(int(i), int(j), block[a, b])

    def get(self, i: int, j: int) -> float:
        if not (0 <= i < self.n_rows and 0 <= j < self.n_cols):
            raise ValueError(f"index ({i}, {j}) out of range for ({self.n_rows}, {self.n_cols})")
        return float(self._cols[j].get(i, 0.0))

    def to_matrix(self) -> CscMatrix:
        ptr = np.zeros(self.n_cols + 1, dtype=np.int64)
        rows, vals = [], []
        for j, col in enumerate(self._cols):
            keys = sorted(col)
            rows.extend(keys)
            vals.extend(col[k] for k in keys)
            ptr[j + 1] = ptr[j] + len(keys)
        return CscMatrix(self.n_rows, self.n_cols, ptr, np.array(rows, dtype=np.int64),
                         np.array(vals, dtype=np.float64), validate=False)

    def __repr__(self) -> str:
        return f"CscBuilder(shape=({self.n_rows}, {self.n_cols}), nnz={self.nnz})"


@dataclass(frozen=True)
class TripletBatch:
    """Element values and positions, one column per triangle (sparse.py:294-329)."""

    rows_per_elem: int
    Ig: np.ndarray
    Jg: np.ndarray
    Kg: np.ndarray

    def __post_init__(self):
        if self.rows_per_elem not in (9, 36):
            raise ValueError(f"rows_per_elem must be 9 or 36, got {self.rows_per_elem}")
        shape = (self.rows_per_elem, self.Ig.shape[1] if self.Ig.ndim == 2 else -1)
        for name in ("Ig", "Jg", "Kg"):
            arr = getattr(self, name)
            if arr.ndim != 2 or tuple(arr.shape) != shape:
                raise ValueError(f"{name} must have shape {shape}, got {tuple(arr.shape)}")

    @property
    def nme(self) -> int:
        return self.Ig.shape[1]

    def flat(self):
        """Column-major 1d arrays: element k occupies slots [k*r, (k+1)*r)."""
        return (np.asarray(self.Ig).ravel(order="F"), np.asarray(self.Jg).ravel(order="F"),
                np.asarray(self.Kg).ravel(order="F"))

    def to_csc(self, n_rows: int, n_cols: int) -> CscMatrix:
        i, j, k = self.flat()
        return csc_from_triplets(i, j, k, n_rows, n_cols)


def write_matrix_market(matrix: CscMatrix, path, threads: int = 0) -> None:
    """Coordinate MatrixMarket, 1-based, values "%.17g", entries in CSC order - the file of
    femasm's write_matrix_market (sparse.py:332-339) byte for byte, written by the library's
    multi-threaded host writer (fa_write_matrix_market; no GPU needed)."""
    import ctypes

    from . import _lib

    cp = np.ascontiguousarray(matrix.col_ptr, dtype=np.int64)
    ri = np.ascontiguousarray(matrix.row_idx, dtype=np.int64)
    va = np.ascontiguousarray(matrix.values, dtype=np.float64)
    rc = _lib.lib().fa_write_matrix_market(os.fsencode(os.fspath(path)), matrix.n_rows, matrix.n_cols,
                                           cp.ctypes.data_as(ctypes.c_void_p), ri.ctypes.data_as(ctypes.c_void_p),
                                           va.ctypes.data_as(ctypes.c_void_p), int(threads))
    if rc != 0:
        raise OSError(_lib.last_error())
