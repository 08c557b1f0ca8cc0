"""GPU parity of the fused OptV2 path (fa_plan_build + fa_assemble via the C ABI) against
the reference: golden full arrays (small meshes), reference digests (BASELINE sizes), the
C oracle (row blocks, edge cases)."""

import numpy as np
import pytest

import paper_1305_3122_b200 as fa
from paper_1305_3122_b200 import _lib
from helpers import assert_same_csc, csc_digests
from oracle import c_oracle
from oracle import femasm_oracle as fo
from paper_1305_3122_b200.meshgen import seeded_square_mesh

pytestmark = pytest.mark.gpu

KINDS = ("mass", "massw", "stiff", "elastic")
SMALL = [f"seeded_n{n}_s{s}" for n in (2, 5, 16) for s in (0, 1)] + ["square_n4", "square_n1", "disk_n4", "disk_n6"]


def plan_assemble(kind, V, C, areas, w=None, lam=1.0, mu=0.5, v0=0, v1=None, recompute=False):
    import torch

    nq, nme = V.shape[0], C.shape[0]
    dev = torch.device("cuda")
    me = torch.from_numpy(np.ascontiguousarray(C, dtype=np.int32)).to(dev)
    q = torch.from_numpy(np.ascontiguousarray(V)).to(dev)
    a = None if recompute else torch.from_numpy(np.ascontiguousarray(areas)).to(dev)
    wd = torch.from_numpy(np.ascontiguousarray(w)).to(dev) if w is not None else None
    plan = fa.AssemblyPlan(nme, nq, v0, nq if v1 is None else v1)
    plan.build(me)
    plan.check_build()
    rowptr, col, val, r = plan.assemble(kind, q=q, areas=a, w=wd, lam=lam, mu=mu)
    return (rowptr.cpu().numpy(), col.cpu().numpy(), val.cpu().numpy()), r


def _case(golden, name, kind):
    V, C = golden[f"{name}/V"], golden[f"{name}/C"]
    w = golden.get(f"{name}/w")
    if w is None:
        w = 1.0 + V[:, 0] * V[:, 0] + V[:, 1] * V[:, 1]
    lm = golden.get(f"{name}/{kind}/lam_mu")
    lam, mu = (float(lm[0]), float(lm[1])) if lm is not None else (1.0, 1.0)
    return V, C, golden[f"{name}/areas"], w, lam, mu


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("name", SMALL)
def test_small_meshes_bitwise(golden, name, kind):
    V, C, areas, w, lam, mu = _case(golden, name, kind)
    got, r = plan_assemble(kind, V, C, areas, w, lam, mu)
    ref = tuple(golden[f"{name}/{kind}/{f}"] for f in ("col_ptr", "row_idx", "values"))
    assert_same_csc(got, ref, f"{name}/{kind}")
    assert r.nnz == len(ref[2])


@pytest.mark.parametrize("kind", ("stiff", "elastic", "mass"))
def test_recomputed_areas_are_bitwise(golden, kind):
    V, C, areas, w, lam, mu = _case(golden, "seeded_n16_s1", kind)
    a, _ = plan_assemble(kind, V, C, areas, w, lam, mu)
    b, _ = plan_assemble(kind, V, C, areas, w, lam, mu, recompute=True)
    assert_same_csc(a, b, kind)


@pytest.mark.parametrize("key", ["C1/s0", "C1/s1", "C1/s2", "EL64/s0", "C2/s0", "C2/s1", "C2/s2"])
def test_reference_digests(digests, key):
    if key not in digests:
        pytest.skip("digest not generated")
    d = digests[key]
    sm = seeded_square_mesh(d["N"], d["seed"])
    areas = c_oracle.areas(sm.vertices, sm.connectivity)
    got, r = plan_assemble(d["kind"], sm.vertices, sm.connectivity, areas, sm.weights, d["lam"], d["mu"])
    assert r.nnz == d["nnz"]
    assert csc_digests(*got) == (d["col_ptr_sha256"], d["row_idx_sha256"], d["values_sha256"])


@pytest.mark.slow
@pytest.mark.parametrize("key", ["C3/s0", "C3/s1", "C3/s2", "C4/s0", "C4/s1", "C4/s2"])
def test_reference_digests_large(digests, key):
    """Full BASELINE sizes (8.4M triangles) against the reference's own output digests;
    C4 seeds differ in how many elasticity positions cancel to exactly 0.0."""
    test_reference_digests(digests, key)


@pytest.mark.slow
@pytest.mark.parametrize("key", ["C5B/s0/G16/b0", "C5B/s0/G8/b7"])
def test_c5_row_block_digest(digests, key):
    """N=8192 (134M triangles): one GPU assembles the vertex-row block of a G-way
    decomposition; the reference digest is the row-block subset assembled by femasm."""
    if key not in digests:
        pytest.skip("digest not generated")
    d = digests[key]
    sm = seeded_square_mesh(d["N"], d["seed"])
    areas = c_oracle.areas(sm.vertices, sm.connectivity)
    got, r = plan_assemble(d["kind"], sm.vertices, sm.connectivity, areas, sm.weights, 1.0, 0.5, d["v0"], d["v1"])
    assert r.nnz == d["nnz"]
    assert csc_digests(*got) == (d["col_ptr_sha256"], d["row_idx_sha256"], d["values_sha256"])


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("blocks", (2, 3, 8))
def test_row_blocks_match_subset_oracle(kind, blocks):
    sm = seeded_square_mesh(24, 3)
    areas = c_oracle.areas(sm.vertices, sm.connectivity)
    full = c_oracle.assemble(kind, sm.vertices, sm.connectivity, areas, sm.weights, 1.0, 0.5)
    rpv = 2 if kind == "elastic" else 1
    cuts = np.linspace(0, sm.nq, blocks + 1).astype(int)
    for v0, v1 in zip(cuts[:-1], cuts[1:]):
        got, _ = plan_assemble(kind, sm.vertices, sm.connectivity, areas, sm.weights, 1.0, 0.5, v0, v1)
        lo, hi = full[0][rpv * v0], full[0][rpv * v1]
        ref = (full[0][rpv * v0: rpv * v1 + 1] - lo, full[1][lo:hi], full[2][lo:hi])
        assert_same_csc(got, ref, f"{kind} [{v0},{v1})")


def fan_mesh(n_spokes, n_rings=2):
    """Star around one hub vertex: degree n_spokes (> 8) exercises the general path."""
    ang = 2 * np.pi * np.arange(n_spokes) / n_spokes
    pts = [np.zeros((1, 2))]
    for r in range(1, n_rings + 1):
        pts.append(np.stack([r * np.cos(ang + 0.1 * r), r * np.sin(ang + 0.1 * r)], axis=1))
    V = np.concatenate(pts)
    tris = []
    for j in range(n_spokes):
        jn = (j + 1) % n_spokes
        tris.append((0, 1 + j, 1 + jn))
        for r in range(1, n_rings):
            a, b = 1 + (r - 1) * n_spokes, 1 + r * n_spokes
            tris.append((a + j, b + j, b + jn))
            tris.append((a + j, b + jn, a + jn))
    C = np.array(tris, dtype=np.int64)
    rng = np.random.default_rng(n_spokes)
    return V, C[rng.permutation(len(C))]


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("spokes", (9, 17, 64))
def test_high_degree_vertices_take_the_general_path(kind, spokes):
    V, C = fan_mesh(spokes)
    areas = fo.triangle_areas(V, C)
    w = np.linspace(0.5, 2.0, V.shape[0])
    ref = fo.assemble_optv2(kind, V, C, areas, w, 2.0, 0.7)
    got, r = plan_assemble(kind, V, C, areas, w, 2.0, 0.7)
    assert r.heavy_rows > 0
    assert_same_csc(got, ref, f"fan{spokes}/{kind}")


def test_deterministic_across_runs():
    sm = seeded_square_mesh(64, 5)
    areas = c_oracle.areas(sm.vertices, sm.connectivity)
    a, _ = plan_assemble("elastic", sm.vertices, sm.connectivity, areas, None, 2.0, 0.7)
    b, _ = plan_assemble("elastic", sm.vertices, sm.connectivity, areas, None, 2.0, 0.7)
    assert_same_csc(a, b, "rerun")


def test_zero_weight_gives_empty_matrix():
    sm = seeded_square_mesh(6, 0)
    areas = fo.triangle_areas(sm.vertices, sm.connectivity)
    got, r = plan_assemble("massw", sm.vertices, sm.connectivity, areas, np.zeros(sm.nq))
    assert r.nnz == 0 and not got[0].any()


def test_degenerate_triangle_reports_first_index():
    V = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0], [2.0, 0.0]])
    C = np.array([[0, 1, 2], [0, 1, 3], [1, 3, 2], [0, 3, 1]])
    areas = fo.triangle_areas(V, C)  # triangles 1 and 3 are collinear
    for kind in ("mass", "stiff", "elastic"):
        _, r = plan_assemble(kind, V, C, areas, None, 1.0, 1.0)
        assert r.degenerate_index == 1, kind
    _, r = plan_assemble("massw", V, C, areas, np.ones(4))
    assert r.degenerate_index == fa._lib.INT64_MAX  # weighted mass never checks (assembly.py:227-243)


def test_connectivity_out_of_range_is_reported():
    import torch

    V = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0]])
    C = np.array([[0, 1, 2], [0, 1, 7]], dtype=np.int32)
    plan = fa.AssemblyPlan(2, 3)
    plan.build(torch.from_numpy(C).cuda())
    with pytest.raises(ValueError, match="out of range"):
        plan.check_build()


def test_repeated_vertex_is_reported():
    """femasm's Mesh rejects a triangle that repeats a vertex id (mesh.py:98-103); a caller of
    the C ABI that skips Mesh gets the plan build's error, and the triangle is left out."""
    import torch

    C = np.array([[0, 1, 2], [1, 3, 3], [2, 2, 0]], dtype=np.int32)
    plan = fa.AssemblyPlan(3, 4)
    plan.build(torch.from_numpy(C).cuda())
    with pytest.raises(ValueError, match="repeated vertex"):
        plan.check_build()
    r = plan._build_res.fetch()
    assert r.repeat_error_pos == 3 * 1 + 2 and r.index_error_pos == _lib.INT64_MAX


def _structured_square(n):
    """Unjittered, unpermuted right-triangle grid: stiffness off-diagonals across the
    hypotenuse sum to exactly zero (Matlab drops them)."""
    n1 = n + 1
    x, y = np.meshgrid(np.linspace(0.0, 1.0, n1), np.linspace(0.0, 1.0, n1))
    V = np.stack([x.ravel(), y.ravel()], axis=1)
    cells = np.arange(n * n)
    iy, ix = np.divmod(cells, n)
    v00 = iy * n1 + ix
    C = np.concatenate([np.stack([v00, v00 + 1, v00 + n1 + 1], 1), np.stack([v00, v00 + n1 + 1, v00 + n1], 1)])
    return V, C


@pytest.mark.parametrize("n", (8, 96, 400))
def test_exact_zero_sums_are_compacted(n):
    """Zero sums stay in the row kernel's symbolic layout and are removed by k_compact; the
    result must equal the reference's dropped pattern (sparse.py:177-179) bit for bit, across
    many buckets (n=400: 161k vertices, 1255 buckets)."""
    V, C = _structured_square(n)
    areas = fo.triangle_areas(V, C)
    ref = c_oracle.assemble("stiff", V, C, areas, None, 1.0, 1.0)
    got, r = plan_assemble("stiff", V, C, areas)
    assert r.dropped > 0
    assert_same_csc(got, ref, f"structured n={n}")


def test_weighted_mass_zero_weights_are_compacted():
    sm = seeded_square_mesh(200, 3)
    areas = fo.triangle_areas(sm.vertices, sm.connectivity)
    w = sm.weights.copy()
    w[::3] = 0.0  # every third vertex weightless: entries among weightless vertices vanish
    w[1::7] = -w[1::7]
    ref = c_oracle.assemble("massw", sm.vertices, sm.connectivity, areas, w, 1.0, 1.0)
    got, r = plan_assemble("massw", sm.vertices, sm.connectivity, areas, w)
    assert r.dropped > 0
    assert_same_csc(got, ref, "massw with zero weights")


@pytest.mark.parametrize("part_log2", (11, 13))
@pytest.mark.parametrize("kind", KINDS)
def test_large_part_general_sort_path(monkeypatch, kind, part_log2):
    """Parts above 1024 vertices (row blocks above 8.4M vertices) are sorted in global memory;
    forced here on a small mesh (with high-degree vertices mixed in) and checked bitwise."""
    monkeypatch.setenv("FEMASM_B200_PART_LOG2", str(part_log2))
    sm = seeded_square_mesh(48, 2)
    V, C = sm.vertices, sm.connectivity
    Vf, Cf = fan_mesh(40)
    V = np.concatenate([V, Vf + 2.0])
    C = np.concatenate([C, Cf + sm.nq])
    areas = fo.triangle_areas(V, C)
    w = 0.5 + np.arange(V.shape[0]) % 7 * 0.25
    ref = c_oracle.assemble(kind, V, C, areas, w, 2.0, 0.7)
    got, _ = plan_assemble(kind, V, C, areas, w, 2.0, 0.7)
    assert_same_csc(got, ref, f"{kind} part_log2={part_log2}")


def hub_part_mesh(n_hubs=1024, spokes=50):
    """n_hubs small fans (hub degree `spokes`) with the hubs numbered first, so the first fine
    part (1024 vertices) holds n_hubs * spokes incidences and every 128-hub bucket overflows
    its shared-memory slots."""
    Vf, Cf = fan_mesh(spokes, n_rings=1)  # hub 0, ring 1..spokes
    nv_f = Vf.shape[0]
    V = np.zeros((n_hubs * nv_f, 2))
    C = []
    for h in range(n_hubs):
        ids = np.concatenate([[h], n_hubs + h * (nv_f - 1) + np.arange(nv_f - 1)])
        V[ids] = Vf + np.array([h, 0.0]) * 3.0
        C.append(ids[Cf])
    C = np.concatenate(C)
    return V, C[np.random.default_rng(1).permutation(len(C))]


@pytest.mark.parametrize("kind", KINDS)
def test_fine_histogram_counter_wrap(monkeypatch, kind):
    """71,680 incidences of one fine part counted by ONE histogram block: its 16-bit shared
    counter wraps (65536 handed to the global fine count and to the block's coarse count).
    Two-level plan forced; bitwise against the oracle."""
    monkeypatch.setenv("FEMASM_B200_COARSE_LOG2", "11")
    monkeypatch.setenv("FEMASM_B200_PLACE_BLOCKS", "1")
    V, C = hub_part_mesh(1024, 70)
    areas = fo.triangle_areas(V, C)
    w = 0.5 + (np.arange(V.shape[0]) % 7) * 0.25
    ref = c_oracle.assemble(kind, V, C, areas, w, 2.0, 0.7)
    got, r = plan_assemble(kind, V, C, areas, w, 2.0, 0.7)
    assert r.heavy_rows > 0
    assert_same_csc(got, ref, f"{kind} wrapped fine counter")


def test_isolated_vertices_have_empty_rows():
    """A vertex no triangle references has no triplet, hence an empty row (reference)."""
    sm = seeded_square_mesh(8, 1)
    V = np.concatenate([sm.vertices, [[5.0, 5.0], [6.0, 6.0]]])
    C = np.asarray(sm.connectivity)
    areas = fo.triangle_areas(V, C)
    w = np.ones(V.shape[0])
    for kind in KINDS:
        ref = c_oracle.assemble(kind, V, C, areas, w, 1.0, 0.5)
        got, _ = plan_assemble(kind, V, C, areas, w, 1.0, 0.5)
        assert_same_csc(got, ref, kind)


@pytest.mark.parametrize("fine_global", (0, 1))
@pytest.mark.parametrize("coarse_log2", (11, 14, 18))
@pytest.mark.parametrize("kind", KINDS)
def test_two_level_plan(monkeypatch, kind, coarse_log2, fine_global):
    """Large row blocks place incidences by coarse part and regroup them by fine part
    (k_part_split); the fine counts come from k_part_hist's shared memory or (more than
    49152 fine parts, forced with fine_global) from global atomics.  Forced here on a small
    mesh and checked bitwise."""
    monkeypatch.setenv("FEMASM_B200_COARSE_LOG2", str(coarse_log2))
    monkeypatch.setenv("FEMASM_B200_FINE_GLOBAL", str(fine_global))
    sm = seeded_square_mesh(70, 4)  # 5041 vertices: 5 fine parts
    areas = fo.triangle_areas(sm.vertices, sm.connectivity)
    ref = c_oracle.assemble(kind, sm.vertices, sm.connectivity, areas, sm.weights, 1.5, 0.6)
    got, _ = plan_assemble(kind, sm.vertices, sm.connectivity, areas, sm.weights, 1.5, 0.6)
    assert_same_csc(got, ref, f"{kind} coarse_log2={coarse_log2}")
    blocks = [(0, 1700), (1700, 3500), (3500, sm.nq)]
    for v0, v1 in blocks:  # row blocks too
        got, _ = plan_assemble(kind, sm.vertices, sm.connectivity, areas, sm.weights, 1.5, 0.6, v0=v0, v1=v1)
        sub = fo.assemble_row_block(kind, sm.vertices, sm.connectivity, areas, sm.weights, 1.5, 0.6, v0, v1)
        assert_same_csc(got, sub, f"{kind} block {v0}:{v1}")


@pytest.mark.parametrize("kind", KINDS)
def test_two_level_sparse_parts(monkeypatch, kind):
    """Vertex ids spread 2048 apart (3.4M mostly isolated vertices): a split round's records
    span more fine parts than its shared-memory window, so some take a cursor each."""
    monkeypatch.setenv("FEMASM_B200_COARSE_LOG2", "14")
    sm = seeded_square_mesh(40, 3)
    spread = 2048
    V = np.zeros((sm.nq * spread, 2))
    V[::spread] = sm.vertices
    C = np.asarray(sm.connectivity, dtype=np.int64) * spread
    areas = fo.triangle_areas(V, C)
    w = 0.5 + np.arange(V.shape[0]) % 7 * 0.25
    ref = c_oracle.assemble(kind, V, C, areas, w, 1.5, 0.6)
    got, _ = plan_assemble(kind, V, C, areas, w, 1.5, 0.6)
    assert_same_csc(got, ref, f"{kind} spread ids")


@pytest.mark.parametrize("kind", KINDS)
def test_vertex_above_bucket_capacity(kind):
    """A hub of degree 1300 overflows its 128-vertex bucket's shared-memory slots (CAPB = 1024):
    every row of that bucket takes the global-memory general path; the plan heap-sorts the
    hub's incidences.  Bitwise against the oracle."""
    V, C = fan_mesh(1300, n_rings=2)
    areas = fo.triangle_areas(V, C)
    w = 0.5 + (np.arange(V.shape[0]) % 5) * 0.3
    ref = c_oracle.assemble(kind, V, C, areas, w, 1.3, 0.4)
    got, r = plan_assemble(kind, V, C, areas, w, 1.3, 0.4)
    assert r.heavy_rows > 0
    assert_same_csc(got, ref, f"{kind} hub 1300")


@pytest.mark.parametrize("block", (None, 0, 1))
@pytest.mark.parametrize("kind", KINDS)
def test_assemble_cold_entry_point(kind, block):
    """fa_assemble_cold (plan build + numeric pass in one call; the weighted mass's triangle
    records on a side stream, or for a row block from the plan's first pass) equals the
    oracle bitwise, repeatedly and after a plain fa_assemble on the same plan (the prepared
    records are consumed once)."""
    import torch
    from paper_1305_3122_b200.device import ResultBlock

    sm = seeded_square_mesh(64, 5)
    areas = fo.triangle_areas(sm.vertices, sm.connectivity)
    v0, v1 = (0, sm.nq) if block is None else [(0, sm.nq // 3), (sm.nq // 3, sm.nq)][block]
    if block is None:
        ref = c_oracle.assemble(kind, sm.vertices, sm.connectivity, areas, sm.weights, 1.0, 0.5)
    else:
        ref = fo.assemble_row_block(kind, sm.vertices, sm.connectivity, areas, sm.weights, 1.0, 0.5, v0, v1)
    dev = torch.device("cuda")
    me = torch.from_numpy(np.ascontiguousarray(sm.connectivity, dtype=np.int32)).to(dev)
    q = torch.from_numpy(sm.vertices).to(dev)
    a = torch.from_numpy(areas).to(dev)
    w = torch.from_numpy(sm.weights).to(dev)
    plan = fa.AssemblyPlan(sm.nme, sm.nq, v0, v1)
    plan.build(me)
    cap = plan.capacity(kind)
    rowptr = torch.empty(plan.rows(kind) + 1, dtype=torch.int64, device=dev)
    col = torch.empty(cap, dtype=torch.int32, device=dev)
    val = torch.empty(cap, dtype=torch.float64, device=dev)
    for it in range(3):
        res = ResultBlock()
        if it == 1:
            plan.assemble_into(kind, q, a, w, 1.0, 0.5, rowptr, col, val, res)
        else:
            plan.assemble_cold_into(me, kind, q, a, w, 1.0, 0.5, rowptr, col, val, res)
        r = res.fetch()
        plan.check_build()
        got = (rowptr.cpu().numpy(), col[: r.nnz].cpu().numpy(), val[: r.nnz].cpu().numpy())
        assert_same_csc(got, ref, f"{kind} cold call {it}")


# ------------------------------------------------------------------------------------------
# the exact timed path of bench.py at BASELINE sizes: fa_assemble_cold from device-resident
# me/q, areas recomputed in the row kernel (stiffness, elasticity) or computed on the device
# (mass, weighted mass; the W records then come from the plan's histogram pass)
# ------------------------------------------------------------------------------------------
def cold_assemble(kind, sm, lam=1.0, mu=0.5, v0=0, v1=None, hash_only=True):
    """bench.py's step (fa_assemble_cold) on seeded mesh `sm`; returns the three CSR digests
    (femasm dtypes) and the fa_result."""
    import torch
    from helpers import csr_digests_device
    from paper_1305_3122_b200.device import ResultBlock

    dev = torch.device("cuda")
    me = torch.from_numpy(np.ascontiguousarray(sm.connectivity, dtype=np.int32)).to(dev)
    q = torch.from_numpy(sm.vertices).to(dev)
    w = torch.from_numpy(sm.weights).to(dev) if kind == "massw" else None
    a = None
    if kind in ("mass", "massw"):
        a = torch.empty(sm.nme, dtype=torch.float64, device=dev)
        ar = ResultBlock()
        _lib.check(_lib.lib().fa_compute_areas(me.data_ptr(), sm.nme, q.data_ptr(), a.data_ptr(), ar.ptr,
                                               _lib.stream_handle()))
    v1 = sm.nq if v1 is None else v1
    plan = fa.AssemblyPlan(sm.nme, sm.nq, v0, v1)
    plan.build(me)
    cap = plan.capacity(kind)
    rowptr = torch.empty(plan.rows(kind) + 1, dtype=torch.int64, device=dev)
    col = torch.empty(cap, dtype=torch.int32, device=dev)
    val = torch.empty(cap, dtype=torch.float64, device=dev)
    res = ResultBlock()
    for _ in range(2):  # twice: the second call reuses the plan's buffers (as the bench's steps)
        plan.assemble_cold_into(me, kind, q if kind in ("stiff", "elastic") else None, a, w, lam, mu,
                                rowptr, col, val, res)
    r = res.fetch()
    plan.check_build()
    assert r.nnz <= cap
    return csr_digests_device(rowptr, col[: r.nnz], val[: r.nnz]), r


@pytest.mark.slow
@pytest.mark.parametrize("key", ["C1/s0", "C1/s1", "C1/s2", "C2/s0", "C2/s1", "C2/s2", "C3/s0", "C4/s0", "C4/s1",
                                 "C4/s2", "EL64/s0"])
def test_timed_path_digests(digests, key):
    """bench.py's exact step against femasm's digests at full BASELINE sizes."""
    d = digests[key]
    sm = seeded_square_mesh(d["N"], d["seed"])
    got, r = cold_assemble(d["kind"], sm, d["lam"] if d["lam"] is not None else 1.0,
                           d["mu"] if d["mu"] is not None else 0.5)
    assert r.nnz == d["nnz"]
    assert got == (d["col_ptr_sha256"], d["row_idx_sha256"], d["values_sha256"])


@pytest.fixture(scope="module")
def c5_mesh():
    return seeded_square_mesh(8192, 0)


@pytest.mark.slow
def test_c5_whole_matrix_digest(digests, c5_mesh):
    """C5 (134M triangles, 470M entries) on one GPU through bench.py's step, against the digest
    of femasm's whole C5 matrix (streamed from its row-block subsets, make_golden.py C5ALL)."""
    d = digests["C5/s0"]
    got, r = cold_assemble("stiff", c5_mesh)
    assert r.nnz == d["nnz"]
    assert got == (d["col_ptr_sha256"], d["row_idx_sha256"], d["values_sha256"])


@pytest.mark.slow
@pytest.mark.parametrize("blk", range(8))
def test_c5_g8_row_blocks(digests, c5_mesh, blk):
    """Every block of the 8-way row split (the multi-GPU decomposition), cold path, against
    femasm's row-block subset digests."""
    d = digests[f"C5B/s0/G8/b{blk}"]
    got, r = cold_assemble("stiff", c5_mesh, v0=d["v0"], v1=d["v1"])
    assert r.nnz == d["nnz"]
    assert got == (d["col_ptr_sha256"], d["row_idx_sha256"], d["values_sha256"])


@pytest.mark.parametrize("kind", KINDS)
def test_reused_plan_with_changed_values(kind):
    """Warm re-assembly: one plan, new numeric inputs each call -
    weights, Lame parameters, coordinates (with recomputed areas) - each bitwise against the
    oracle for those inputs."""
    import torch
    from paper_1305_3122_b200.device import ResultBlock

    sm = seeded_square_mesh(40, 6)
    dev = torch.device("cuda")
    me = torch.from_numpy(np.ascontiguousarray(sm.connectivity, dtype=np.int32)).to(dev)
    plan = fa.AssemblyPlan(sm.nme, sm.nq)
    plan.build(me)
    rng = np.random.default_rng(11)
    for it in range(3):
        V = sm.vertices.copy()
        interior = (V[:, 0] > 0) & (V[:, 0] < 1) & (V[:, 1] > 0) & (V[:, 1] < 1)
        V[interior] += rng.uniform(-0.002, 0.002, (int(interior.sum()), 2)) * it
        w = rng.uniform(0.5, 2.0, sm.nq) if it else sm.weights
        lam, mu = [(1.0, 0.5), (2.0, 0.7), (0.3, 1.9)][it]
        areas = fo.triangle_areas(V, sm.connectivity)
        ref = c_oracle.assemble(kind, V, sm.connectivity, areas, w, lam, mu)
        q = torch.from_numpy(V).to(dev)
        a = None if kind in ("stiff", "elastic") else torch.from_numpy(areas).to(dev)
        wd = torch.from_numpy(w).to(dev)
        rowptr, col, val, r = plan.assemble(kind, q=q, areas=a, w=wd, lam=lam, mu=mu)
        assert_same_csc((rowptr.cpu().numpy(), col.cpu().numpy(), val.cpu().numpy()), ref, f"{kind} call {it}")


def test_row_block_capacity_after_build_on_a_side_stream():
    """fa_plan_capacity reads the row block's incidence count on the stream the build ran on
    (a non-blocking stream is not ordered with the legacy default stream)."""
    import torch

    sm = seeded_square_mesh(64, 3)
    me = torch.from_numpy(sm.connectivity.astype(np.int32)).cuda()
    ref = fa.AssemblyPlan(sm.nme, sm.nq, 500, 2500)
    ref.build(me)
    torch.cuda.synchronize()
    want = ref.capacity("stiff")
    side = torch.cuda.Stream()
    for _ in range(3):
        plan = fa.AssemblyPlan(sm.nme, sm.nq, 500, 2500)
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            plan.build(me, stream=side)
            assert plan.capacity("stiff") == want
