"""Small assemblies through every library kernel family, for compute-sanitizer
(tests/test_sanitizer.py): cold and warm OptV2 for the four kinds on a seeded mesh, a mesh with
a high-degree hub (general path, bucket overflow), a two-level plan with a row block, exact-zero
sums (k_compact), the general triplet path and the element-loop strategies."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import numpy as np
import torch

import paper_1305_3122_b200 as fa
from paper_1305_3122_b200.device import ResultBlock
from paper_1305_3122_b200.meshgen import seeded_square_mesh

dev = torch.device("cuda")


def run(V, C, w, v0=0, v1=None):
    me = torch.from_numpy(np.ascontiguousarray(C, dtype=np.int32)).to(dev)
    q = torch.from_numpy(np.ascontiguousarray(V)).to(dev)
    a = torch.from_numpy(fa.compute_areas(V, C)).to(dev)
    wd = torch.from_numpy(np.ascontiguousarray(w)).to(dev)
    plan = fa.AssemblyPlan(C.shape[0], V.shape[0], v0, V.shape[0] if v1 is None else v1)
    for kind in ("mass", "massw", "stiff", "elastic"):
        plan.build(me)
        cap = plan.capacity(kind)
        rowptr = torch.empty(plan.rows(kind) + 1, dtype=torch.int64, device=dev)
        col = torch.empty(cap, dtype=torch.int32, device=dev)
        val = torch.empty(cap, dtype=torch.float64, device=dev)
        res = ResultBlock()
        plan.assemble_cold_into(me, kind, q, None if kind in ("stiff", "elastic") else a, wd, 1.0, 0.5, rowptr, col,
                                val, res)
        plan.assemble_into(kind, q, a, wd, 1.0, 0.5, rowptr, col, val, res)
        torch.cuda.synchronize()


sm = seeded_square_mesh(12, 1)
run(sm.vertices, sm.connectivity, sm.weights)
run(sm.vertices, sm.connectivity, sm.weights, 40, 120)
from test_gpu_parity import fan_mesh  # noqa: E402

V, C = fan_mesh(1100, n_rings=1)  # hub above a bucket's capacity
run(V, C, np.ones(V.shape[0]))
os.environ["FEMASM_B200_COARSE_LOG2"] = "11"
sm2 = seeded_square_mesh(50, 2)
run(sm2.vertices, sm2.connectivity, sm2.weights, 100, 2000)
del os.environ["FEMASM_B200_COARSE_LOG2"]
sq = fa.generate_unit_square_mesh(6)  # exact-zero stiffness sums: k_compact moves segments
fa.assemble(sq, fa.MatrixKind.STIFFNESS, fa.Strategy.OPTV2)
fa.assemble(sq, fa.MatrixKind.STIFFNESS, fa.Strategy.CLASSICAL)
fa.assemble(sq, fa.MatrixKind.ELASTIC, fa.Strategy.OPTV1, params=fa.ElasticParams(1.0, 0.5))
rng = np.random.default_rng(0)
fa.csc_from_triplets(rng.integers(0, 50, 3000), rng.integers(0, 40, 3000), rng.standard_normal(3000), 50, 40)
torch.cuda.synchronize()
print("sanitize case done")
