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


class _Slot:
    """Device inputs/outputs and pinned host outputs of one in-flight step."""

    def __init__(self, torch, dev, kind, nq, nme, rows, needs_q, recompute_areas):
        self.me = torch.empty((nme, 3), dtype=torch.int32, device=dev)
        self.q = torch.empty((nq, 2), dtype=torch.float64, device=dev) if needs_q else None
        self.areas = None if recompute_areas else torch.empty(nme, dtype=torch.float64, device=dev)
        self.w = torch.empty(nq, dtype=torch.float64, device=dev) if kind == "massw" else None
        self.rowptr = torch.empty(rows + 1, dtype=torch.int64, device=dev)
        self.res = ResultBlock()
        self.h_rowptr = torch.empty(rows + 1, dtype=torch.int64, pin_memory=True)
        self.bres = torch.empty(_lib.RESULT_WORDS, dtype=torch.int64, device=dev)  # the plan build's block
        self.h_res = torch.empty(2 * _lib.RESULT_WORDS, dtype=torch.int64, pin_memory=True)
        self.col = self.val = self.h_col = self.h_val = None
        self.ev_me, self.ev_in, self.ev_comp, self.ev_meta, self.ev_out = (torch.cuda.Event() for _ in range(5))
        self.ticket = None  # step occupying the slot, until its result is collected
        self.used = False


class HostAssembler:
    """Reusable end-to-end assembler for one (kind, nq, nme, row block).

    ``run(me, q, areas, w, lam, mu)`` takes host arrays (pinned torch CPU tensors for
    overlap-free DMA, or numpy), copies them to the device, builds the plan, assembles and
    copies rowptr/col/val back into pinned host tensors.  Returns (rowptr, col, val, nnz): host
    tensors (views of the pinned buffers, valid until the slot is reused) and the entry count.

    ``submit`` / ``result`` split a call in two so that a stream of problems of one size
    pipelines over ``depth`` buffer slots: the host->device copy of step i+1 and its plan +
    assembly run while the device->host copy of step i is in flight (PCIe is full duplex; the
    copies use side streams, the kernels the caller's stream; the entry arrays of step i go on
    a stream of their own so they never queue behind step i+1's kernels).  ``run`` = submit +
    result.
    The result blocks of the last collected step are ``last_result`` (assembly: nnz, first
    degenerate triangle) and ``last_build_result`` (plan build: first out-of-range vertex id).
    """

    def __init__(self, kind: str, nq: int, nme: int, row_begin: int = 0, row_end: int | None = None,
                 recompute_areas: bool = False, depth: int = 2):
        torch = require_cuda()
        if depth < 1:
            raise ValueError("depth must be >= 1")
        self.kind = kind
        self.nq, self.nme = int(nq), int(nme)
        self.recompute_areas = bool(recompute_areas)
        dev = device()
        self.plan = AssemblyPlan(nme, nq, row_begin, row_end)
        self.rows = self.plan.rows(kind)
        needs_q = kind in ("stiff", "elastic") or recompute_areas
        self._slots = [_Slot(torch, dev, kind, self.nq, self.nme, self.rows, needs_q, self.recompute_areas)
                       for _ in range(depth)]
        self._h2d = torch.cuda.Stream()
        self._meta = torch.cuda.Stream()  # row pointers + result blocks (waits for the kernels)
        self._d2h = torch.cuda.Stream()   # entry arrays (issued by result(), never queued behind a later step)
        self._next = 0
        self._cap = None
        self.last_result = self.last_build_result = None

    def _ensure_capacity(self, s: _Slot):
        torch = require_cuda()
        if self._cap is None:
            self._cap = max(self.plan.capacity(self.kind), 1)
        if s.col is None:
            dev = device()
            s.col = torch.empty(self._cap, dtype=torch.int32, device=dev)
            s.val = torch.empty(self._cap, dtype=torch.float64, device=dev)
            s.h_col = torch.empty(self._cap, dtype=torch.int32, pin_memory=True)
            s.h_val = torch.empty(self._cap, dtype=torch.float64, pin_memory=True)

    def submit(self, me, q=None, areas=None, w=None, lam=0.0, mu=0.0, stream=None) -> int:
        """Queue one step (asynchronous); returns its ticket for ``result``."""
        torch = require_cuda()
        st = stream or torch.cuda.current_stream()
        ticket = self._next
        s = self._slots[ticket % len(self._slots)]
        if s.ticket is not None:  # the slot's previous step must be collected first
            self.result(s.ticket)
        self._next += 1

        def h2d(dst, src):
            if dst is None:
                return
            t = src if isinstance(src, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(src))
            dst.copy_(t.view(dst.shape), non_blocking=True)

        # inputs: after the kernels that last read this slot; the connectivity first (the plan
        # needs only it), the numeric inputs while the plan is built
        if s.used:
            self._h2d.wait_event(s.ev_comp)
        else:
            self._h2d.wait_stream(st)
        with torch.cuda.stream(self._h2d):
            h2d(s.me, me)
            s.ev_me.record(self._h2d)
            h2d(s.q, q)
            h2d(s.areas, areas)
            h2d(s.w, w)
            s.ev_in.record(self._h2d)
        with torch.cuda.stream(st):
            st.wait_event(s.ev_me)
            self.plan.build(s.me, st)
            s.bres.copy_(self.plan._build_res.dev)  # stream-ordered: before the next build resets it
            self._ensure_capacity(s)
            st.wait_event(s.ev_in)
            self.plan.assemble_into(self.kind, s.q, s.areas, s.w, lam, mu, s.rowptr, s.col, s.val, s.res, st)
            s.ev_comp.record(st)
        self._meta.wait_event(s.ev_comp)
        with torch.cuda.stream(self._meta):  # sizes known on the host: row pointers + result blocks
            s.h_res[: _lib.RESULT_WORDS].copy_(s.res.dev, non_blocking=True)
            s.h_res[_lib.RESULT_WORDS:].copy_(s.bres, non_blocking=True)
            s.h_rowptr.copy_(s.rowptr, non_blocking=True)
            s.ev_meta.record(self._meta)
        s.ticket = ticket
        s.used = True
        return ticket

    def result(self, ticket: int):
        """Wait for step ``ticket``; returns (rowptr, col, val, nnz) host views of its slot."""
        torch = require_cuda()
        s = self._slots[ticket % len(self._slots)]
        if s.ticket != ticket:
            raise ValueError(f"step {ticket} is not in flight (slot holds {s.ticket})")
        s.ev_meta.synchronize()
        r = _lib.result_from_words(s.h_res[: _lib.RESULT_WORDS])
        rb = _lib.result_from_words(s.h_res[_lib.RESULT_WORDS:])
        self.last_result, self.last_build_result = r, rb
        nnz = int(r.nnz)
        if nnz > self._cap:  # the capacity is sized once, from the first step's plan
            s.ticket = None
            raise RuntimeError(f"assembly needs {nnz} entries, the buffers hold {self._cap}: the row block's "
                               "incidence count grew; use a new HostAssembler for this connectivity")
        self._d2h.wait_event(s.ev_comp)
        with torch.cuda.stream(self._d2h):  # entry arrays: nnz is known now
            s.h_col[:nnz].copy_(s.col[:nnz], non_blocking=True)
            s.h_val[:nnz].copy_(s.val[:nnz], non_blocking=True)
            s.ev_out.record(self._d2h)
        s.ev_out.synchronize()
        s.ticket = None
        return s.h_rowptr, s.h_col[:nnz], s.h_val[:nnz], nnz

    def run(self, me, q=None, areas=None, w=None, lam=0.0, mu=0.0, stream=None):
        return self.result(self.submit(me, q, areas, w, lam, mu, stream))

    def bytes_h2d(self) -> int:
        s = self._slots[0]
        return sum(int(t.numel() * t.element_size()) for t in (s.me, s.q, s.areas, s.w) if t is not None)


def _host_assemble(kind, nq, nme, me, q=None, areas=None, w=None, lam=0.0, mu=0.0) -> CscMatrix:
    me = connectivity_int32(np.asarray(me).reshape(int(nme), 3))
    a = HostAssembler(kind, nq, nme, depth=1)
    rowptr, col, val, nnz = a.run(me, q, areas, w, lam, mu)
    r = a.last_result
    if a.last_build_result.index_error_pos != _lib.INT64_MAX:
        raise ValueError("connectivity index out of range [0, nq)")
    if a.last_build_result.repeat_error_pos != _lib.INT64_MAX:
        raise ValueError("triangle with repeated vertex indices")
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
