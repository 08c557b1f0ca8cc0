"""Per-block phase timeline of the row kernel (experiment build with -DFA_EXP_TIMELINE)."""
import ctypes, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_1305_3122_b200 as fa
from paper_1305_3122_b200 import _lib
from paper_1305_3122_b200.device import ResultBlock
from paper_1305_3122_b200.meshgen import seeded_square_mesh, BASELINE_CONFIGS
cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
NAMES = (sys.argv[2].split(",") if len(sys.argv) > 2 else ["p1", "p2", "p3", "p4", "p5"])
kind, n, lam, mu = BASELINE_CONFIGS[cfg]
sm = seeded_square_mesh(n, 0)
dev = torch.device("cuda")
me = torch.from_numpy(sm.connectivity.astype(np.int32)).to(dev)
q = torch.from_numpy(sm.vertices).to(dev)
a = torch.from_numpy(fa.compute_areas(sm.vertices, sm.connectivity)).to(dev)
w = torch.from_numpy(sm.weights).to(dev) if kind == "massw" else None
plan = fa.AssemblyPlan(sm.nme, sm.nq); plan.build(me)
cap = plan.capacity(kind)
rowptr = torch.empty(plan.rows(kind) + 1, dtype=torch.int64, device=dev)
col = torch.empty(cap, dtype=torch.int32, device=dev); val = torch.empty(cap, dtype=torch.float64, device=dev)
res = ResultBlock()
for _ in range(3):
    plan.build(me); plan.assemble_into(kind, q, a, w, lam or 0.0, mu or 0.0, rowptr, col, val, res)
torch.cuda.synchronize()
lib = _lib.lib()
lib.fa_debug_timeline.argtypes = [ctypes.c_void_p, ctypes.c_int64]
nb = min(16384, (sm.nq + 127) // 128)
buf = np.zeros(16384 * 6, dtype=np.uint64)
lib.fa_debug_timeline(buf.ctypes.data, buf.size)
t = buf[: nb * 6].reshape(nb, 6).astype(np.int64)
t0 = t[:, 0].min()
t = t - t0
d = np.diff(t, axis=1)
print("kernel span us", (t[:, 5].max()) / 1e3)
for i, name in enumerate(NAMES):
    print(f"{name:16s} mean {d[:, i].mean()/1e3:7.2f} us  p50 {np.median(d[:, i])/1e3:7.2f}  p90 {np.percentile(d[:, i], 90)/1e3:7.2f}")
print("block duration mean", (t[:, 5] - t[:, 0]).mean() / 1e3, "us; start spread", t[:, 0].max() / 1e3)
conc = np.zeros(200)
for s_, e_ in zip(t[:, 0], t[:, 5]):
    conc[int(s_ // 2000): int(e_ // 2000) + 1] += 1
print("concurrent blocks (2us bins, first 40):", conc[:40].astype(int).tolist())
