"""Randomised GPU parity: unstructured and irregular meshes the fixed suites do not hold
(Delaunay triangulations of random point sets with vertex degrees up to ~15, duplicated and
mirrored triangles, unused vertices, row blocks cut at random rows, plans of every depth),
each assembled through fa_plan_build + fa_assemble and through fa_assemble_cold (areas given
and recomputed) and compared bitwise with the C oracle on the same arrays.

Reference semantics exercised: assembly.py:400-416 (_assemble_batched), sparse.py:140-189
(csc_from_triplets: stable order, sequential sums, exact-zero drop), mesh.py:62-65 (areas)."""

import numpy as np
import pytest

import paper_1305_3122_b200 as fa
from helpers import assert_same_csc
from oracle import c_oracle
from paper_1305_3122_b200.meshgen import seeded_square_mesh

pytestmark = pytest.mark.gpu

KINDS = ("mass", "massw", "stiff", "elastic")


def delaunay_mesh(rng, npts):
    """Delaunay triangulation of random points (clustered, so degrees vary widely), counter-
    clockwise triangles, vertex and triangle numbering permuted."""
    from scipy.spatial import Delaunay

    pts = rng.random((npts, 2))
    k = npts // 4
    pts[:k] = 0.5 + 0.02 * rng.standard_normal((k, 2))  # a dense cluster: small areas, high degrees
    tri = Delaunay(pts).simplices.astype(np.int64)
    a, b, c = pts[tri[:, 0]], pts[tri[:, 1]], pts[tri[:, 2]]
    cross = (b[:, 0] - a[:, 0]) * (c[:, 1] - a[:, 1]) - (c[:, 0] - a[:, 0]) * (b[:, 1] - a[:, 1])
    tri[cross < 0] = tri[cross < 0][:, [0, 2, 1]]
    perm = rng.permutation(npts)
    inv = np.empty(npts, dtype=np.int64)
    inv[perm] = np.arange(npts)
    V = pts[perm]
    C = inv[tri][rng.permutation(len(tri))]
    return V, C


def irregular(rng, V, C):
    """Oddities femasm accepts: triangles listed twice (their triplets add up), clockwise
    copies (areas are absolute values), vertices no triangle references (empty rows)."""
    nme = C.shape[0]
    dup = C[rng.integers(0, nme, size=max(1, nme // 50))]
    cw = C[rng.integers(0, nme, size=max(1, nme // 50))][:, [0, 2, 1]]
    C2 = np.concatenate([C, dup, cw])
    C2 = C2[rng.permutation(len(C2))]
    extra = rng.random((int(rng.integers(1, 40)), 2))
    V2 = np.concatenate([V, extra])
    # the unused vertices get ids spread over the range, not only the top
    perm = rng.permutation(V2.shape[0])
    inv = np.empty_like(perm)
    inv[perm] = np.arange(perm.size)
    return V2[perm], inv[C2]


def gpu_both_paths(kind, V, C, areas, w, lam, mu, v0, v1, recompute):
    """(plan + assemble, cold) CSR triples on the GPU for rows [v0, v1)."""
    import torch
    from paper_1305_3122_b200.device import ResultBlock

    dev = torch.device("cuda")
    nq, nme = V.shape[0], C.shape[0]
    me = torch.from_numpy(np.ascontiguousarray(C, dtype=np.int32)).to(dev)
    q = torch.from_numpy(np.ascontiguousarray(V)).to(dev)
    a = None if recompute else torch.from_numpy(np.ascontiguousarray(areas)).to(dev)
    wd = torch.from_numpy(np.ascontiguousarray(w)).to(dev) if kind == "massw" else None
    plan = fa.AssemblyPlan(nme, nq, v0, v1)
    plan.build(me)
    plan.check_build()
    rowptr, col, val, r = plan.assemble(kind, q=q, areas=a, w=wd, lam=lam, mu=mu)
    warm = (rowptr.cpu().numpy(), col.cpu().numpy(), val.cpu().numpy())
    cap = plan.capacity(kind)
    rp = torch.empty(plan.rows(kind) + 1, dtype=torch.int64, device=dev)
    cc = torch.empty(cap, dtype=torch.int32, device=dev)
    vv = torch.empty(cap, dtype=torch.float64, device=dev)
    res = ResultBlock()
    plan.assemble_cold_into(me, kind, q, a, wd, lam, mu, rp, cc, vv, res)
    rc = res.fetch()
    plan.check_build()
    cold = (rp.cpu().numpy(), cc[: rc.nnz].cpu().numpy(), vv[: rc.nnz].cpu().numpy())
    return warm, cold, r


def check_case(kind, V, C, w, lam, mu, v0, v1, recompute, what):
    areas = c_oracle.areas(V, C)
    if kind == "massw":
        recompute = False  # the weighted mass always takes areas
    rpv = 2 if kind == "elastic" else 1
    ref = c_oracle.assemble(kind, V, C, areas, w, lam, mu, rpv * v0, rpv * v1)
    warm, cold, r = gpu_both_paths(kind, V, C, areas, w, lam, mu, v0, v1, recompute)
    assert_same_csc(warm, ref, f"{what} plan+assemble")
    assert_same_csc(cold, ref, f"{what} cold")
    return r


@pytest.mark.parametrize("seed", range(16))
def test_delaunay_meshes_bitwise(seed):
    rng = np.random.default_rng(1000 + seed)
    npts = int(rng.integers(50, 6000)) if seed < 12 else int(rng.integers(20000, 80000))
    V, C = delaunay_mesh(rng, npts)
    if seed % 2:
        V, C = irregular(rng, V, C)
    nq = V.shape[0]
    w = rng.uniform(0.5, 2.0, nq)
    heavy = 0
    for kind in KINDS:
        lam, mu = float(rng.uniform(0.1, 3.0)), float(rng.uniform(0.1, 3.0))
        cuts = sorted({0, nq, *(int(x) for x in rng.integers(0, nq + 1, size=2))})
        for v0, v1 in [(0, nq)] + list(zip(cuts[:-1], cuts[1:])):
            if v0 == v1:
                continue
            r = check_case(kind, V, C, w, lam, mu, v0, v1, bool(rng.integers(0, 2)),
                           f"delaunay seed {seed} npts {npts} {kind} rows [{v0},{v1})")
            heavy += r.heavy_rows
    assert heavy > 0  # clustered Delaunay meshes have vertices of degree > 8


@pytest.mark.parametrize("seed", range(12))
def test_square_meshes_random_blocks_and_plan_depths(monkeypatch, seed):
    """The benchmark's mesh family at random sizes, rows cut at random, with the plan forced
    through its two-level and global-sort variants."""
    rng = np.random.default_rng(2000 + seed)
    n = int(rng.integers(3, 200))
    sm = seeded_square_mesh(n, int(rng.integers(0, 1000)))
    V, C = sm.vertices, sm.connectivity
    if seed % 4 == 3:
        V, C = irregular(rng, V, C)
    nq = V.shape[0]
    w = rng.uniform(0.5, 2.0, nq)
    if seed % 2:
        monkeypatch.setenv("FEMASM_B200_COARSE_LOG2", str(int(rng.integers(11, 15))))
    if seed % 4 == 2:
        monkeypatch.setenv("FEMASM_B200_PART_LOG2", "12")
    for kind in KINDS:
        v0 = int(rng.integers(0, nq))
        v1 = int(rng.integers(v0 + 1, nq + 1))
        for a, b in ((0, nq), (v0, v1)):
            check_case(kind, V, C, w, 1.0, 0.5, a, b, bool(rng.integers(0, 2)),
                       f"square n {n} seed {seed} {kind} rows [{a},{b})")
