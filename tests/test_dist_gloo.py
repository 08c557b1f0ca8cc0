"""Host-side multi-rank logic of the row-block decomposition (paper_1305_3122_b200.dist) on
CPU with the gloo backend, world_size 2 and 3: row blocks, the nnz allgather that yields the
global row offsets, and the gather to rank 0, with the row-block subset oracle standing in
for each rank's GPU kernel.  The stitched matrix must equal the full assembly bit for bit."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import femasm_oracle as fo
from paper_1305_3122_b200.dist import RowBlockCsr, gather_to_rank0, global_offsets, row_blocks, stitch_blocks
from paper_1305_3122_b200.meshgen import seeded_square_mesh


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, kind, out_q):
    import torch

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sm = seeded_square_mesh(12, 7)
        areas = fo.triangle_areas(sm.vertices, sm.connectivity)
        v0, v1 = row_blocks(sm.nq, world)[rank]
        ptr, idx, vals = fo.assemble_row_block(kind, sm.vertices, sm.connectivity, areas, sm.weights, 2.0, 0.7, v0, v1)
        offset, total = global_offsets(int(ptr[-1]))
        rpv = 2 if kind == "elastic" else 1
        stitched = gather_to_rank0(torch.from_numpy(ptr), torch.from_numpy(idx.astype(np.int32)),
                                   torch.from_numpy(vals), rpv * v0, rpv * sm.nq)
        out_q.put((rank, offset, total, int(ptr[-1]),
                   None if stitched is None else tuple(np.asarray(a) for a in stitched)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("kind", ["stiff", "elastic"])
def test_row_block_exchange_with_gloo(world, kind):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    results.sort()
    sm = seeded_square_mesh(12, 7)
    areas = fo.triangle_areas(sm.vertices, sm.connectivity)
    full = fo.assemble_optv2(kind, sm.vertices, sm.connectivity, areas, sm.weights, 2.0, 0.7)
    running = 0
    for rank, offset, total, local, _ in results:
        assert offset == running and total == len(full[2])
        running += local
    rowptr, col, val = results[0][4]
    assert np.array_equal(rowptr, full[0])
    assert np.array_equal(col.astype(np.int64), full[1])
    assert np.array_equal(val, full[2])


def test_row_blocks_cover_and_balance():
    for nq, world in [(10, 3), (66049, 8), (5, 8), (1, 1)]:
        blocks = row_blocks(nq, world)
        assert blocks[0][0] == 0 and blocks[-1][1] == nq
        assert all(a[1] == b[0] for a, b in zip(blocks, blocks[1:]))
        sizes = [b - a for a, b in blocks]
        assert max(sizes) - min(sizes) <= 1


def test_stitch_rejects_gaps():
    b0 = RowBlockCsr(0, np.array([0, 1]), np.array([0]), np.array([1.0]))
    b2 = RowBlockCsr(2, np.array([0, 1]), np.array([2]), np.array([1.0]))
    with pytest.raises(ValueError):
        stitch_blocks([b0, b2], 3)
    rowptr, col, val = stitch_blocks([b0, RowBlockCsr(1, np.array([0, 0]), np.zeros(0, int), np.zeros(0))], 2)
    assert rowptr.tolist() == [0, 1, 1]
