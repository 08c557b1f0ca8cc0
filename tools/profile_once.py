"""Run one config's cold assembly a few times (for ncu captures)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import paper_1305_3122_b200 as fa
from paper_1305_3122_b200.device import ResultBlock
from paper_1305_3122_b200.meshgen import seeded_square_mesh, BASELINE_CONFIGS

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
G = int(sys.argv[3]) if len(sys.argv) > 3 else 1  # optional: rank 0's row block of a G-way split
kind, n, lam, mu = BASELINE_CONFIGS[cfg]
sm = seeded_square_mesh(n, 0)
dev = torch.device("cuda")
me = torch.from_numpy(sm.connectivity.astype(np.int32)).to(dev)
q = torch.from_numpy(sm.vertices).to(dev)
a = torch.from_numpy(fa.compute_areas(sm.vertices, sm.connectivity)).to(dev)
import os
if os.environ.get("RECOMPUTE", "1") == "1" and kind in ("stiff", "elastic"):
    a = None  # bench mode: areas recomputed in the row kernel
w = torch.from_numpy(sm.weights).to(dev) if kind == "massw" else None
from paper_1305_3122_b200.dist import row_blocks
v0, v1 = row_blocks(sm.nq, G)[0]
plan = fa.AssemblyPlan(sm.nme, sm.nq, v0, v1)
plan.build(me)
cap = plan.capacity(kind)
rowptr = torch.empty(plan.rows(kind) + 1, dtype=torch.int64, device=dev)
col = torch.empty(cap, dtype=torch.int32, device=dev)
val = torch.empty(cap, dtype=torch.float64, device=dev)
res = ResultBlock()
for _ in range(reps):
    plan.build(me)
    plan.assemble_into(kind, q, a, w, lam or 0.0, mu or 0.0, rowptr, col, val, res)
torch.cuda.synchronize()
print(cfg, "nnz", res.fetch().nnz)
