"""Device timing of the reference-API building blocks off the fused path (development tool):
compute_areas, batch_kg_*, build_ig_jg_p1, batch_gradients and the general csc_from_triplets on
the Kg/Ig/Jg triplets of a BASELINE config (CUDA events, L2 flushed before each launch, median
of REPS).  Prints a markdown table with algorithmic bytes and GB/s.

usage: python tools/batch_time.py [CONFIG] [REPS]"""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_1305_3122_b200 as fa
from paper_1305_3122_b200 import _lib
from paper_1305_3122_b200.device import ResultBlock
from paper_1305_3122_b200.meshgen import BASELINE_CONFIGS, seeded_square_mesh

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
kind, n, lam, mu = BASELINE_CONFIGS[cfg]
sm = seeded_square_mesh(n, 0)
dev = torch.device("cuda")
L = _lib.lib()
st = _lib.stream_handle()
me = torch.from_numpy(sm.connectivity.astype(np.int32)).to(dev)
q = torch.from_numpy(sm.vertices).to(dev)
nme, nq = sm.nme, sm.nq
kcode = _lib.KIND_CODES[kind]
r = 36 if kind == "elastic" else 9
areas = torch.empty(nme, dtype=torch.float64, device=dev)
kg = torch.empty(r * nme, dtype=torch.float64, device=dev)
ig = torch.empty(r * nme, dtype=torch.int32, device=dev)
jg = torch.empty(r * nme, dtype=torch.int32, device=dev)
g6 = torch.empty(6 * nme, dtype=torch.float64, device=dev)
w = torch.from_numpy(sm.weights).to(dev) if kind == "massw" else None
res = ResultBlock()
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
P = lambda t: t.data_ptr() if t is not None else None  # noqa: E731


def timed(fn):
    ts = []
    for i in range(reps + 1):
        flush.zero_()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        if i:
            ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


rows = []
t = timed(lambda: _lib.check(L.fa_compute_areas(P(me), nme, P(q), P(areas), res.ptr, st), "areas"))
rows.append(("compute_areas (`k_areas`)", t, nme * (12 + 8) + nq * 16))
t = timed(lambda: _lib.check(L.fa_element_kg(kcode, P(me), nme, P(q), P(areas), P(w), lam or 1.0, mu or 0.5, P(kg),
                                             res.ptr, st), "kg"))
rows.append((f"batch_kg ({kind}, `k_element_kg`)", t, nme * (12 + 8 + 8 * r) + nq * 16))
t = timed(lambda: _lib.check(L.fa_build_ig_jg(1 if kind == "elastic" else 0, P(me), nme, P(ig), P(jg), st), "igjg"))
rows.append(("build_ig_jg (`k_ig_jg`)", t, nme * (12 + 8 * r)))
t = timed(lambda: _lib.check(L.fa_batch_gradients(P(me), nme, P(q), P(areas), P(g6), res.ptr, st), "grad"))
rows.append(("batch_gradients (`k_gradients`)", t, nme * (12 + 8 + 48) + nq * 16))
# general sparse(): the reference's TripletBatch (Ig, Jg, Kg raveled) -> CSC
ln = r * nme
ri, ci = ig.to(torch.int64), jg.to(torch.int64)
ndof = 2 * nq if kind == "elastic" else nq
ws_b = L.fa_triplets_workspace(ln, ndof, ndof)
ws = torch.empty(ws_b, dtype=torch.uint8, device=dev)
cp = torch.empty(ndof + 1, dtype=torch.int64, device=dev)
ro = torch.empty(ln, dtype=torch.int64, device=dev)
vo = torch.empty(ln, dtype=torch.float64, device=dev)
t = timed(lambda: _lib.check(L.fa_triplets_to_csc(P(ri), P(ci), P(kg), ln, ndof, ndof, P(cp), P(ro), P(vo), P(ws), ws_b,
                                                  res.ptr, st), "triplets"))
nnz = int(res.fetch().nnz)
rows.append((f"csc_from_triplets ({ln:,} triplets -> {nnz:,} entries)", t, ln * 24 + (ndof + 1) * 8 + nnz * 16))
print(f"| {cfg} kernel | ms | algorithmic bytes | GB/s |")
print("|---|---|---|---|")
for name, ms, b in rows:
    print(f"| {name} | {ms:.3f} | {b / 1e6:.1f} MB | {b / (ms * 1e-3) / 1e9:.0f} |")
