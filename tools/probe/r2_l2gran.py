"""Row-kernel time at C5 (recomputed areas, bench mode) under cudaLimitMaxL2FetchGranularity
32 / 64 / 128 (development probe)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np
import torch
from cuda.bindings import runtime as rt
import paper_1305_3122_b200 as fa
from paper_1305_3122_b200 import _lib
from paper_1305_3122_b200.device import ResultBlock
from paper_1305_3122_b200.meshgen import seeded_square_mesh, BASELINE_CONFIGS

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
kind, n, lam, mu = BASELINE_CONFIGS[cfg]
sm = seeded_square_mesh(n, 0)
dev = torch.device("cuda")
me = torch.from_numpy(sm.connectivity.astype(np.int32)).to(dev)
q = torch.from_numpy(sm.vertices).to(dev)
w = torch.from_numpy(sm.weights).to(dev) if kind == "massw" else None
a = None
if kind in ("mass", "massw"):
    a = torch.empty(sm.nme, dtype=torch.float64, device=dev)
    rb = ResultBlock()
    _lib.lib().fa_compute_areas(me.data_ptr(), sm.nme, q.data_ptr(), a.data_ptr(), rb.ptr, _lib.stream_handle())
plan = fa.AssemblyPlan(sm.nme, sm.nq)
plan.build(me)
cap = plan.capacity(kind)
rowptr = torch.empty(plan.rows(kind) + 1, dtype=torch.int64, device=dev)
col = torch.empty(cap, dtype=torch.int32, device=dev)
val = torch.empty(cap, dtype=torch.float64, device=dev)
res = ResultBlock()
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
for gran in (128, 64, 32):
    err, = rt.cudaDeviceSetLimit(rt.cudaLimit.cudaLimitMaxL2FetchGranularity, gran)
    err2, got = rt.cudaDeviceGetLimit(rt.cudaLimit.cudaLimitMaxL2FetchGranularity)
    tb, tn = [], []
    for i in range(5):
        flush.zero_()
        e[0].record()
        plan.build(me)
        e[1].record()
        plan.assemble_into(kind, q if kind in ("stiff", "elastic") else None, a, w, lam or 1.0, mu or 0.5, rowptr, col, val, res)
        e[2].record()
        torch.cuda.synchronize()
        if i >= 2:
            tb.append(e[0].elapsed_time(e[1])); tn.append(e[1].elapsed_time(e[2]))
    print(f"{cfg} L2 fetch granularity {got} ({err}): build {np.median(tb):.3f} ms numeric {np.median(tn):.3f} ms nnz {res.fetch().nnz}", flush=True)
