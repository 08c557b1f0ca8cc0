"""Quick device timing of plan build + numeric assembly per config (development tool)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import paper_1305_3122_b200 as fa
from paper_1305_3122_b200.device import ResultBlock
from paper_1305_3122_b200.meshgen import seeded_square_mesh, BASELINE_CONFIGS

def run(cfg, reps=10, recompute=True):
    kind, n, lam, mu = BASELINE_CONFIGS[cfg]
    sm = seeded_square_mesh(n, 0)
    dev = torch.device("cuda")
    me = torch.from_numpy(sm.connectivity.astype(np.int32)).to(dev)
    q = torch.from_numpy(sm.vertices).to(dev)
    areas = fa.compute_areas(sm.vertices, sm.connectivity)
    a = None if (recompute and kind in ("stiff", "elastic")) else torch.from_numpy(areas).to(dev)
    w = torch.from_numpy(sm.weights).to(dev) if kind == "massw" else None
    plan = fa.AssemblyPlan(sm.nme, sm.nq)
    plan.build(me); plan.check_build()
    cap = plan.capacity(kind)
    rowptr = torch.empty(plan.rows(kind) + 1, dtype=torch.int64, device=dev)
    col = torch.empty(cap, dtype=torch.int32, device=dev)
    val = torch.empty(cap, dtype=torch.float64, device=dev)
    res = ResultBlock()
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    tb, tn = [], []
    for i in range(reps + 3):
        flush.zero_()
        e[0].record()
        plan.build(me)
        e[1].record()
        plan.assemble_into(kind, q, a, w, lam or 0.0, mu or 0.0, rowptr, col, val, res)
        e[2].record()
        torch.cuda.synchronize()
        if i >= 3:
            tb.append(e[0].elapsed_time(e[1])); tn.append(e[1].elapsed_time(e[2]))
    r = res.fetch()
    tb, tn = np.median(tb), np.median(tn)
    print(f"{cfg} {kind} N={n} nme={sm.nme} nnz={r.nnz} heavy={r.heavy_rows} build={tb*1e3:.1f}us numeric={tn*1e3:.1f}us "
          f"cold={(tb+tn)*1e3:.1f}us tri/s={sm.nme/((tb+tn)*1e-3):.3e} warm tri/s={sm.nme/(tn*1e-3):.3e}", flush=True)

for cfg in sys.argv[1:] or ["C1", "C2", "C3", "C4"]:
    run(cfg)
