"""Multi-GPU OptV2 by vertex-row blocks.

Rank g owns the matrix rows of the vertices [v_g, v_{g+1}); a CSR row depends only on the
triangles incident to its vertex, so every rank assembles its block independently (its plan
scans all of the connectivity and keeps only its incidences) and no cross-GPU sum exists.
The one data exchange is the row-offset allgather: each rank contributes its local nnz and
obtains the global offset of its first row (NCCL over NVLink on GPUs, gloo in the CPU
tests).  An optional gather to rank 0 assembles the global CSR there (grouped point-to-point
transfers; NCCL has no gather primitive).

The reference has no distribution at all (single-threaded numpy, femasm/bench.py:81); the
row-block decomposition is verified bit-exact against the full assembly through the
row-block subset oracle (oracle/femasm_oracle.py: assemble_row_block).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["row_blocks", "global_offsets", "RowBlockCsr", "stitch_blocks", "DistributedAssembler"]


def row_blocks(nq: int, world_size: int) -> list[tuple[int, int]]:
    """Contiguous, balanced vertex-row blocks [v0, v1) for each rank (random numbering
    balances incidences across equal vertex ranges)."""
    if world_size < 1:
        raise ValueError("world_size must be >= 1")
    cuts = [(nq * g) // world_size for g in range(world_size + 1)]
    return [(cuts[g], cuts[g + 1]) for g in range(world_size)]


def global_offsets(local_nnz: int, group=None) -> tuple[int, int]:
    """All-gather every rank's local nnz; return (this rank's global entry offset, total nnz).
    Uses the default process group (NCCL on GPUs, gloo on CPU)."""
    import torch
    import torch.distributed as dist

    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    mine = torch.tensor([int(local_nnz)], dtype=torch.int64, device=dev)
    world = dist.get_world_size(group)
    parts = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(parts, mine, group=group)
    counts = [int(p.item()) for p in parts]
    rank = dist.get_rank(group)
    return sum(counts[:rank]), sum(counts)


@dataclass
class RowBlockCsr:
    """One rank's share of the global CSR: local row pointers (starting at 0) of rows
    [row0, row0 + n_rows), global column ids, values, and the global entry offset."""

    row0: int
    rowptr: np.ndarray
    col: np.ndarray
    val: np.ndarray
    entry_offset: int = 0

    @property
    def n_rows(self) -> int:
        return len(self.rowptr) - 1

    @property
    def nnz(self) -> int:
        return int(self.rowptr[-1])


def stitch_blocks(blocks: list[RowBlockCsr], n_rows: int):
    """Concatenate row blocks (in row order) into global (rowptr int64, col, val)."""
    blocks = sorted(blocks, key=lambda b: b.row0)
    rowptr = np.zeros(n_rows + 1, dtype=np.int64)
    cols, vals = [], []
    base = 0
    expect = 0
    for b in blocks:
        if b.row0 != expect:
            raise ValueError(f"row blocks are not contiguous at row {expect}")
        rowptr[b.row0: b.row0 + b.n_rows + 1] = np.asarray(b.rowptr, dtype=np.int64) + base
        cols.append(np.asarray(b.col))
        vals.append(np.asarray(b.val))
        base += b.nnz
        expect = b.row0 + b.n_rows
    if expect != n_rows:
        raise ValueError(f"row blocks cover {expect} of {n_rows} rows")
    return rowptr, np.concatenate(cols) if cols else np.zeros(0, np.int32), np.concatenate(vals) if vals else np.zeros(0)


class DistributedAssembler:
    """Row-block OptV2 on this rank's GPU.  Inputs are full (device) arrays of the mesh;
    the plan covers this rank's vertex rows only."""

    def __init__(self, kind: str, nq: int, nme: int, rank: int, world_size: int):
        from .plan import KIND_ROWS_PER_VERTEX, AssemblyPlan

        self.kind = kind
        self.nq, self.nme = int(nq), int(nme)
        self.rank, self.world = int(rank), int(world_size)
        self.v0, self.v1 = row_blocks(self.nq, self.world)[self.rank]
        self.rpv = KIND_ROWS_PER_VERTEX[kind]
        self.plan = AssemblyPlan(self.nme, self.nq, self.v0, self.v1)

    @property
    def row0(self) -> int:
        return self.v0 * self.rpv

    def assemble(self, me_dev, q=None, areas=None, w=None, lam=0.0, mu=0.0, exchange=True):
        """Plan build + fused assembly of this rank's rows; with `exchange`, the NCCL
        allgather of local nnz gives the global entry offset.  Returns (rowptr, col, val,
        entry_offset, total_nnz, fa_result)."""
        from . import _lib
        from .mesh import DegenerateTriangleError

        self.plan.build(me_dev)
        self.plan.check_build()  # out-of-range / repeated vertex ids: the reference's ValueError
        rowptr, col, val, r = self.plan.assemble(self.kind, q=q, areas=areas, w=w, lam=lam, mu=mu)
        if r.degenerate_index != _lib.INT64_MAX:
            k = int(r.degenerate_index)
            area = float(areas[k].item()) if areas is not None else 0.0
            raise DegenerateTriangleError(k, area)
        offset, total = (0, int(r.nnz))
        if exchange and self.world > 1:
            offset, total = global_offsets(int(r.nnz))
        return rowptr, col, val, offset, total, r


def gather_to_rank0(rowptr, col, val, row0: int, n_rows_global: int, group=None):
    """Optional gather of every rank's CSR block to rank 0 (point-to-point sends; NCCL has
    no gather).  Returns the global (rowptr, col, val) on rank 0, None elsewhere."""
    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    dev = rowptr.device
    meta = torch.tensor([row0, rowptr.numel() - 1, col.numel()], dtype=torch.int64, device=dev)
    metas = [torch.empty_like(meta) for _ in range(world)]
    dist.all_gather(metas, meta, group=group)
    if rank != 0:
        ops = [dist.P2POp(dist.isend, t.contiguous(), 0, group) for t in (rowptr, col, val)]
        for req in dist.batch_isend_irecv(ops):
            req.wait()
        return None
    blocks_t = []
    ops = []
    for g in range(world):
        r0, nr, nz = (int(x) for x in metas[g].tolist())
        if g == 0:
            blocks_t.append((r0, rowptr, col, val))
            continue
        rp = torch.empty(nr + 1, dtype=rowptr.dtype, device=dev)
        cc = torch.empty(nz, dtype=col.dtype, device=dev)
        vv = torch.empty(nz, dtype=val.dtype, device=dev)
        ops += [dist.P2POp(dist.irecv, t, g, group) for t in (rp, cc, vv)]
        blocks_t.append((r0, rp, cc, vv))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    blocks = [RowBlockCsr(r0, rp.cpu().numpy(), cc.cpu().numpy(), vv.cpu().numpy()) for r0, rp, cc, vv in blocks_t]
    return stitch_blocks(blocks, n_rows_global)
