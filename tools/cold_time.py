"""Cold step through fa_plan_build + fa_assemble vs fa_assemble_cold, eager and graph-replayed
(development tool): python tools/cold_time.py [CFG [G RANK]] - with G, RANK: that rank's row block
of a G-way row-block decomposition (bench.py's split), timed alone on this GPU."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import paper_1305_3122_b200 as fa
from paper_1305_3122_b200.device import ResultBlock
from paper_1305_3122_b200.meshgen import seeded_square_mesh, BASELINE_CONFIGS

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
G = int(sys.argv[2]) if len(sys.argv) > 2 else 1
rank = int(sys.argv[3]) if len(sys.argv) > 3 else 0
kind, n, lam, mu = BASELINE_CONFIGS[cfg]
sm = seeded_square_mesh(n, 0)
dev = torch.device("cuda")
me = torch.from_numpy(sm.connectivity.astype(np.int32)).to(dev)
q = torch.from_numpy(sm.vertices).to(dev)
a = torch.from_numpy(fa.compute_areas(sm.vertices, sm.connectivity)).to(dev)
if kind in ("stiff", "elastic"):  # recomputed from q, as assemble() does for an exact-area Mesh
    a = None
w = torch.from_numpy(sm.weights).to(dev) if kind == "massw" else None
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1305_3122_b200.dist import row_blocks  # noqa: E402
v0, v1 = row_blocks(sm.nq, G)[rank]
plan = fa.AssemblyPlan(sm.nme, sm.nq, v0, v1)
plan.build(me)
cap = plan.capacity(kind)
rowptr = torch.empty(plan.rows(kind) + 1, dtype=torch.int64, device=dev)
col = torch.empty(cap, dtype=torch.int32, device=dev)
val = torch.empty(cap, dtype=torch.float64, device=dev)
res = ResultBlock()
flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev)
s = torch.cuda.Stream()


def split_step():
    plan.build(me, stream=s)
    plan.assemble_into(kind, q, a, w, lam or 0.0, mu or 0.0, rowptr, col, val, res, stream=s)


def cold_step():
    plan.assemble_cold_into(me, kind, q, a, w, lam or 0.0, mu or 0.0, rowptr, col, val, res, stream=s)


def timed(fn, graph, reps=30):
    if graph:
        with torch.cuda.stream(s):
            fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            fn()
        run = g.replay
    else:
        run = fn
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for i in range(reps + 3):
        flush.zero_()
        torch.cuda.synchronize()
        with torch.cuda.stream(s):
            e0.record(s)
            run()
            e1.record(s)
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(e0.elapsed_time(e1) * 1e3)
    r = res.fetch()
    return np.median(ts), r.nnz


for name, fn in (("build+assemble", split_step), ("assemble_cold", cold_step)):
    for graph in (False, True):
        t, nnz = timed(fn, graph)
        print(f"{cfg} G={G} rank={rank} {name:16s} graph={graph!s:5s} {t:8.1f} us  nnz={nnz}  "
              f"tri/s (this block's share of the mesh) {sm.nme / G / (t * 1e-6):.3e}", flush=True)
