"""Per-rank cold step of the row-block decomposition, each rank's block
timed alone on this GPU (the pool gives one GPU per call): for G in (1, 2, 4, 8) every rank's
fa_assemble_cold (plan build of its rows + row kernel, CUDA-graph replay, L2 flushed before
each step), the max over ranks, and the implied G-GPU speed-up of the compute (the NCCL nnz
allgather, 8 bytes per rank, is not included).  Writes a markdown table to stdout.

usage: python tools/rank_times.py [CONFIG] [REPS]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_1305_3122_b200 as fa
from paper_1305_3122_b200.device import ResultBlock
from paper_1305_3122_b200.dist import row_blocks
from paper_1305_3122_b200.meshgen import BASELINE_CONFIGS, seeded_square_mesh

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
GS = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [1, 2, 4, 8]
kind, n, lam, mu = BASELINE_CONFIGS[cfg]
sm = seeded_square_mesh(n, 0)
dev = torch.device("cuda")
me = torch.from_numpy(sm.connectivity.astype(np.int32)).to(dev)
q = torch.from_numpy(sm.vertices).to(dev)
a = None
if kind in ("mass", "massw"):
    a = torch.from_numpy(fa.compute_areas(sm.vertices, sm.connectivity)).to(dev)
w = torch.from_numpy(sm.weights).to(dev) if kind == "massw" else None
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
s = torch.cuda.Stream()
rows = []
for G in GS:
    times = []
    for rank, (v0, v1) in enumerate(row_blocks(sm.nq, G)):
        plan = fa.AssemblyPlan(sm.nme, sm.nq, v0, v1)
        plan.build(me)
        cap = plan.capacity(kind)
        rowptr = torch.empty(plan.rows(kind) + 1, dtype=torch.int64, device=dev)
        col = torch.empty(cap, dtype=torch.int32, device=dev)
        val = torch.empty(cap, dtype=torch.float64, device=dev)
        res = ResultBlock()
        qq = q if kind in ("stiff", "elastic") else None

        def step():
            plan.assemble_cold_into(me, kind, qq, a, w, lam or 1.0, mu or 0.5, rowptr, col, val, res, stream=s)

        with torch.cuda.stream(s):
            step()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            step()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts = []
        for i in range(reps + 2):
            flush.zero_()
            torch.cuda.synchronize()
            with torch.cuda.stream(s):
                e0.record(s)
                g.replay()
                e1.record(s)
            torch.cuda.synchronize()
            if i >= 2:
                ts.append(e0.elapsed_time(e1))
        times.append(float(np.median(ts)))
        del plan, g, rowptr, col, val
        torch.cuda.empty_cache()
    rows.append((G, times))
t1 = rows[0][1][0]
print(f"| G | per-rank cold step (ms) | max over ranks (ms) | implied speed-up | efficiency |")
print("|---|---|---|---|---|")
for G, ts in rows:
    mx = max(ts)
    print(f"| {G} | {', '.join(f'{t:.2f}' for t in ts)} | {mx:.2f} | {t1 / mx:.2f}x | {t1 / mx / G * 100:.0f} % |", flush=True)
