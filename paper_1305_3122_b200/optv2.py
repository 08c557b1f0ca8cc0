"""Paper-level OptV2 entry points on host buffers (arXiv 1305.3122, PAPER.md:938, :1402,
:1513, :2091):

    MassAssemblingP1OptV2(nq, nme, me, areas)
    MassWAssemblingP1OptV2(nq, nme, me, areas, Tw)
    StiffAssemblingP1OptV2(nq, nme, q, me, areas)
    StiffElasAssemblingP1OptV2(nq, nme, q, me, areas, lam, mu)

(with the femasm conventions: ``q`` (nq, 2) float64, ``me`` (nme, 3) 0-based, ``areas``
(nme,)).  Each call is the complete end-to-end path a CPU caller sees: host->device copy of
the inputs, plan build (symbolic), fused numeric assembly, device->host copy of the CSR.
``HostAssembler`` keeps the device/pinned buffers of one problem size for repeated calls;
it is what the e2e leg of bench.py times.  The base / OptV1 variants of the paper are the
same computation here (``*AssemblingP1base`` and ``*AssemblingP1OptV1`` alias OptV2).
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .device import ResultBlock, connectivity_int32, device, require_cuda
from .plan import AssemblyPlan
from .sparse import CscMatrix

__all__ = [
    "HostAssembler",
    "MassAssemblingP1OptV2",
    "MassWAssemblingP1OptV2",
    "StiffAssemblingP1OptV2",
    "StiffElasAssemblingP1OptV2",
    "MassAssemblingP1OptV1",
    "MassWAssemblingP1OptV1",
    "StiffAssemblingP1OptV1",
    "StiffElasAssemblingP1OptV1",
    "MassAssemblingP1base",
    "MassWAssemblingP1base",
    "StiffAssemblingP1base",
    "StiffElasAssemblingP1base",
]


class HostAssembler:
    """Reusable end-to-end assembler for one (kind, nq, nme, row block).

    ``run(me, q, areas, w, lam, mu)`` takes host arrays (pinned torch CPU tensors for
    overlap-free DMA, or numpy), copies them to the device, builds the plan, assembles and
    copies rowptr/col/val back into pinned host tensors.  Returns (rowptr, col, val) host
    tensors (views of the pinned buffers, valid until the next run) and the fa_result.
    """

    def __init__(self, kind: str, nq: int, nme: int, row_begin: int = 0, row_end: int | None = None,
                 recompute_areas: bool = False):
        torch = require_cuda()
        self.kind = kind
        self.nq, self.nme = int(nq), int(nme)
        self.recompute_areas = bool(recompute_areas)
        dev = device()
        self.plan = AssemblyPlan(nme, nq, row_begin, row_end)
        self.me = torch.empty((self.nme, 3), dtype=torch.int32, device=dev)
        needs_q = kind in ("stiff", "elastic") or recompute_areas
        self.q = torch.empty((self.nq, 2), dtype=torch.float64, device=dev) if needs_q else None
        self.areas = None if recompute_areas else torch.empty(self.nme, dtype=torch.float64, device=dev)
        self.w = torch.empty(self.nq, dtype=torch.float64, device=dev) if kind == "massw" else None
        self.rows = self.plan.rows(kind)
        self.rowptr = torch.empty(self.rows + 1, dtype=torch.int64, device=dev)
        self.res = ResultBlock()
        self._cap = None
        self.h_rowptr = torch.empty(self.rows + 1, dtype=torch.int64, pin_memory=True)
        self.h_nnz = torch.empty(1, dtype=torch.int64, pin_memory=True)
        self._side = None

    def _ensure_capacity(self):
        torch = require_cuda()
        if self._cap is None:
            cap = self.plan.capacity(self.kind)
            dev = device()
            self.col = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
            self.val = torch.empty(max(cap, 1), dtype=torch.float64, device=dev)
            self.h_col = torch.empty(max(cap, 1), dtype=torch.int32, pin_memory=True)
            self.h_val = torch.empty(max(cap, 1), dtype=torch.float64, pin_memory=True)
            self._cap = cap

    def run(self, me, q=None, areas=None, w=None, lam=0.0, mu=0.0, stream=None):
        torch = require_cuda()
        st = stream or torch.cuda.current_stream()

        def h2d(dst, src):
            if dst is None:
                return
            s = src if isinstance(src, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(src))
            dst.copy_(s.view(dst.shape), non_blocking=True)

        # the connectivity first (the plan needs only it); the numeric inputs travel on a side
        # stream while the plan is built
        if self._side is None:
            self._side = torch.cuda.Stream()
        self._side.wait_stream(st)
        with torch.cuda.stream(self._side):
            h2d(self.q, q)
            h2d(self.areas, areas)
            h2d(self.w, w)
        with torch.cuda.stream(st):
            h2d(self.me, me)
            self.plan.build(self.me, st)
            self._ensure_capacity()
            st.wait_stream(self._side)
            self.plan.assemble_into(self.kind, self.q, self.areas, self.w, lam, mu, self.rowptr, self.col,
                                    self.val, self.res, st)
            self.h_rowptr.copy_(self.rowptr, non_blocking=True)
            self.h_nnz.copy_(self.rowptr[-1:], non_blocking=True)
        st.synchronize()
        nnz = int(self.h_nnz[0])
        with torch.cuda.stream(st):
            self.h_col[:nnz].copy_(self.col[:nnz], non_blocking=True)
            self.h_val[:nnz].copy_(self.val[:nnz], non_blocking=True)
        st.synchronize()
        return self.h_rowptr, self.h_col[:nnz], self.h_val[:nnz], nnz

    def bytes_h2d(self) -> int:
        return sum(int(t.numel() * t.element_size()) for t in (self.me, self.q, self.areas, self.w) if t is not None)


def _host_assemble(kind, nq, nme, me, q=None, areas=None, w=None, lam=0.0, mu=0.0) -> CscMatrix:
    me = connectivity_int32(np.asarray(me).reshape(int(nme), 3))
    a = HostAssembler(kind, nq, nme)
    rowptr, col, val, nnz = a.run(me, q, areas, w, lam, mu)
    r = a.res.fetch()
    if r.index_error_pos != _lib.INT64_MAX:
        raise ValueError("connectivity index out of range [0, nq)")
    if r.degenerate_index != _lib.INT64_MAX:
        from .mesh import DegenerateTriangleError

        k = int(r.degenerate_index)
        raise DegenerateTriangleError(k, float(np.asarray(areas)[k]))
    n = int(nq) * (2 if kind == "elastic" else 1)
    return CscMatrix(n, n, rowptr.numpy().copy(), col.numpy().astype(np.int64), val.numpy().copy(), validate=False)


def MassAssemblingP1OptV2(nq, nme, me, areas) -> CscMatrix:
    return _host_assemble("mass", nq, nme, me, areas=areas)


def MassWAssemblingP1OptV2(nq, nme, me, areas, Tw) -> CscMatrix:
    return _host_assemble("massw", nq, nme, me, areas=areas, w=Tw)


def StiffAssemblingP1OptV2(nq, nme, q, me, areas) -> CscMatrix:
    return _host_assemble("stiff", nq, nme, me, q=q, areas=areas)


def StiffElasAssemblingP1OptV2(nq, nme, q, me, areas, lam, mu) -> CscMatrix:
    return _host_assemble("elastic", nq, nme, me, q=q, areas=areas, lam=lam, mu=mu)


MassAssemblingP1OptV1 = MassAssemblingP1base = MassAssemblingP1OptV2
MassWAssemblingP1OptV1 = MassWAssemblingP1base = MassWAssemblingP1OptV2
StiffAssemblingP1OptV1 = StiffAssemblingP1base = StiffAssemblingP1OptV2
StiffElasAssemblingP1OptV1 = StiffElasAssemblingP1base = StiffElasAssemblingP1OptV2
