"""Assembly plans: the symbolic half of OptV2 (incidence structure) owned by the library.

A plan covers one block of vertex rows [row_begin, row_end) of one mesh connectivity; the
whole mesh is (0, nq).  ``AssemblyPlan.assemble`` runs the fused numeric kernel and returns
device CSR arrays (rowptr int64 local, col int32 global, val f64).  Reference counterpart:
the index builders + sort of OptV2 (assembly.py:162-192, sparse.py:164-168), which the
reference recomputes on every call; a plan can be reused (warm assembly).
"""

from __future__ import annotations

import ctypes

from . import _lib
from .device import ResultBlock, device, require_cuda

KIND_ROWS_PER_VERTEX = {"mass": 1, "massw": 1, "stiff": 1, "elastic": 2}


class AssemblyPlan:
    def __init__(self, nme: int, nq: int, row_begin: int = 0, row_end: int | None = None):
        require_cuda()
        self.nme = int(nme)
        self.nq = int(nq)
        self.row_begin = int(row_begin)
        self.row_end = self.nq if row_end is None else int(row_end)
        handle = ctypes.c_void_p()
        rc = _lib.lib().fa_plan_create(ctypes.byref(handle), self.nme, self.nq, self.row_begin, self.row_end)
        _lib.check(rc, "fa_plan_create")
        self._h = handle
        self._me = None
        self._build_res = ResultBlock()
        self._capacity = {}

    @property
    def handle(self):
        return self._h

    def build(self, me_dev, stream=None) -> None:
        """(Re)build the incidence structure from device connectivity (nme, 3) int32."""
        self._me = me_dev  # keep alive: the weighted-mass numeric pass reads it (fa_plan_build contract)
        self._capacity.clear()
        rc = _lib.lib().fa_plan_build(self._h, me_dev.data_ptr(), self._build_res.ptr, _lib.stream_handle(stream))
        _lib.check(rc, "fa_plan_build")

    def check_build(self, stream=None) -> None:
        """Raise the reference's ValueError for an invalid connectivity (mesh.py:95-103).
        Synchronises `stream` (the one the build ran on) first."""
        if stream is not None:
            stream.synchronize()
        r = self._build_res.fetch()
        if r.index_error_pos != _lib.INT64_MAX:
            raise ValueError("connectivity index out of range [0, nq)")
        if r.repeat_error_pos != _lib.INT64_MAX:
            raise ValueError("triangle with repeated vertex indices")

    def rows(self, kind: str) -> int:
        return (self.row_end - self.row_begin) * KIND_ROWS_PER_VERTEX[kind]

    def capacity(self, kind: str) -> int:
        if kind not in self._capacity:
            cap = ctypes.c_int64()
            rc = _lib.lib().fa_plan_capacity(self._h, _lib.KIND_CODES[kind], ctypes.byref(cap))
            _lib.check(rc, "fa_plan_capacity")
            self._capacity[kind] = int(cap.value)
        return self._capacity[kind]

    def assemble_into(self, kind, q, areas, w, lam, mu, rowptr, col, val, result: ResultBlock, stream=None) -> None:
        """Launch the numeric assembly into caller buffers (asynchronous)."""
        rc = _lib.lib().fa_assemble(
            self._h, _lib.KIND_CODES[kind], _lib.ptr(q), _lib.ptr(areas), _lib.ptr(w),
            float(lam), float(mu), rowptr.data_ptr(), col.data_ptr(), val.data_ptr(),
            int(col.numel()), result.ptr, _lib.stream_handle(stream),
        )
        _lib.check(rc, "fa_assemble")

    def assemble_cold_into(self, me_dev, kind, q, areas, w, lam, mu, rowptr, col, val, result: ResultBlock,
                           stream=None) -> None:
        """Plan build + numeric assembly in one asynchronous call (fa_assemble_cold): the cold
        OptV2; the weighted mass's triangle records are computed concurrently with the build.
        Build errors: check_build()."""
        self._me = me_dev
        self._capacity.clear()
        rc = _lib.lib().fa_assemble_cold(
            self._h, me_dev.data_ptr(), _lib.KIND_CODES[kind], _lib.ptr(q), _lib.ptr(areas), _lib.ptr(w),
            float(lam), float(mu), rowptr.data_ptr(), col.data_ptr(), val.data_ptr(), int(col.numel()),
            self._build_res.ptr, result.ptr, _lib.stream_handle(stream),
        )
        _lib.check(rc, "fa_assemble_cold")

    def assemble(self, kind, q=None, areas=None, w=None, lam=0.0, mu=0.0, stream=None):
        """Allocate outputs, assemble, synchronise; returns (rowptr, col, val, fa_result)."""
        torch = require_cuda()
        dev = device()
        n_rows = self.rows(kind)
        cap = self.capacity(kind)
        rowptr = torch.empty(n_rows + 1, dtype=torch.int64, device=dev)
        col = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
        val = torch.empty(max(cap, 1), dtype=torch.float64, device=dev)
        res = ResultBlock()
        self.assemble_into(kind, q, areas, w, lam, mu, rowptr, col, val, res, stream)
        if stream is not None:  # the result block is read on the current stream below
            stream.synchronize()
        r = res.fetch()  # synchronises
        if r.nnz > cap:
            raise RuntimeError(f"assembly produced {r.nnz} entries but the plan's capacity is {cap}")
        return rowptr, col[: r.nnz], val[: r.nnz], r

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            _lib.lib().fa_plan_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
