"""The drop-in API on the GPU: batch kernels, general csc_from_triplets, assemble() through
Mesh for every strategy, the paper-level entry points and the hand-off converters — each
against the reference golden fixtures or the oracle (reference tests cited per case)."""

import numpy as np
import pytest

import paper_1305_3122_b200 as fa
from helpers import assert_same_csc
from oracle import femasm_oracle as fo

pytestmark = pytest.mark.gpu

SEEDED = [f"seeded_n{n}_s{s}" for n in (5, 16) for s in (0, 1)]


def mesh_of(golden, name):
    return fa.Mesh(golden[f"{name}/V"], golden[f"{name}/C"])


@pytest.mark.parametrize("name", SEEDED)
def test_batch_kernels_bitwise(golden, name):
    mesh = mesh_of(golden, name)
    assert np.array_equal(mesh.areas.view(np.int64), golden[f"{name}/areas"].view(np.int64))
    w = golden[f"{name}/w"]
    for got, key in (
        (fa.batch_kg_mass(mesh.areas), "kg_mass"),
        (fa.batch_kg_mass_weighted(mesh, fa.WeightField.samples(w)), "kg_massw"),
        (fa.batch_kg_stiff(mesh), "kg_stiff"),
        (fa.batch_kg_elastic(mesh, fa.ElasticParams(1.0, 0.5)), "kg_elastic"),
    ):
        ref = golden[f"{name}/{key}"]
        assert got.shape == ref.shape
        assert np.array_equal(got.view(np.int64), ref.view(np.int64)), key
    g = fa.batch_gradients(mesh)
    assert np.array_equal(np.concatenate([g.g1, g.g2, g.g3]), golden[f"{name}/grad"])


def test_index_batches_reference_examples():
    # test_assembly.py:50-53, :70-74
    ig, jg = fa.build_ig_jg_p1(np.array([[5, 7, 9]]))
    assert ig[:, 0].tolist() == [5, 7, 9, 5, 7, 9, 5, 7, 9]
    assert jg[:, 0].tolist() == [5, 5, 5, 7, 7, 7, 9, 9, 9]
    ig, jg = fa.build_ig_jg_p1_vector(np.array([[0, 1, 2]]))
    assert ig[:, 0].tolist() == [0, 1, 2, 3, 4, 5] * 6
    assert jg[:, 0].tolist() == [d for d in range(6) for _ in range(6)]
    conn = fa.generate_unit_square_mesh(3).connectivity
    ig, jg = fa.build_ig_jg_p1(conn)
    rig, rjg = fo.index_pattern(conn, vector=False)
    assert np.array_equal(ig, rig) and np.array_equal(jg, rjg)


def test_value_batches_reference_examples():
    # test_assembly.py:122-135, :151-165 and test_elements.py:70-77
    kg = fa.batch_kg_mass(np.array([0.5]))
    expect = [1 / 12, 1 / 24, 1 / 24, 1 / 24, 1 / 12, 1 / 24, 1 / 24, 1 / 24, 1 / 12]
    assert np.abs(kg[:, 0] - expect).max() <= 1e-16
    kg = fa.batch_kg_mass(np.array([6.0, 12.0]))
    assert kg[[0, 4, 8], 0].tolist() == [1.0, 1.0, 1.0] and kg[[0, 4, 8], 1].tolist() == [2.0, 2.0, 2.0]
    mesh = fa.Mesh(np.array([[0.0, 0.0], [30.0, 0.0], [0.0, 2.0]]), np.array([[0, 1, 2]]))
    kg = fa.batch_kg_mass_weighted(mesh, fa.WeightField.samples([1.0, 2.0, 3.0]))
    assert kg[:, 0].tolist() == [8.0, 4.5, 5.0, 4.5, 10.0, 5.5, 5.0, 5.5, 12.0]
    unit = fa.Mesh(np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0]]), np.array([[0, 1, 2]]))
    kg = fa.batch_kg_stiff(unit)
    assert kg[:, 0].tolist() == [1.0, -0.5, -0.5, -0.5, 0.5, 0.0, -0.5, 0.0, 0.5]
    e = fa.elem_mass_weighted(30.0, 1.0, 2.0, 3.0)
    assert (e[0, 0], e[0, 1], e[0, 2], e[1, 1], e[1, 2], e[2, 2]) == (8.0, 4.5, 5.0, 10.0, 5.5, 12.0)


def test_degenerate_batch_raises_with_index():
    with pytest.raises(fa.DegenerateTriangleError) as exc:
        fa.batch_kg_mass(np.array([1.0, 0.0, 0.0]))
    assert exc.value.index == 1
    with pytest.raises(fa.DegenerateTriangleError) as exc:
        fa.Mesh(np.array([[0.0, 0.0], [1.0, 0.0], [2.0, 0.0]]), np.array([[0, 1, 2]]))
    assert exc.value.index == 0


def test_csc_from_triplets_reference_examples():
    # test_sparse.py:16-57
    a = fa.csc_from_triplets([0, 1, 2, 2, 0, 1], [0, 1, 1, 2, 3, 3], [1.0, 5.0, 1.0, 2.0, 6.0, 4.0], 3, 4)
    assert a.values.tolist() == [1, 5, 1, 2, 6, 4]
    assert a.row_idx.tolist() == [0, 1, 2, 2, 0, 1] and a.col_ptr.tolist() == [0, 1, 3, 4, 6]
    assert fa.csc_from_triplets([0, 0], [0, 0], [2.0, 3.0], 1, 1).values.tolist() == [5.0]
    assert fa.csc_from_triplets([0, 0], [0, 0], [2.0, -2.0], 1, 1).nnz == 0
    b = fa.csc_from_triplets([0, 1], [0, 0], [0.0, 1.0], 2, 1)
    assert b.nnz == 1 and b.get(0, 0) == 0.0 and b.get(1, 0) == 1.0
    e = fa.csc_from_triplets([], [], [], 3, 3)
    assert e.nnz == 0 and e.get(2, 2) == 0.0
    with pytest.raises(ValueError, match="length"):
        fa.csc_from_triplets([0, 1], [0], [1.0, 2.0], 2, 2)
    with pytest.raises(ValueError, match="position 1"):
        fa.csc_from_triplets([0, 5], [0, 0], [1.0, 2.0], 3, 3)
    with pytest.raises(ValueError, match="column"):
        fa.csc_from_triplets([0, 0], [0, -1], [1.0, 2.0], 3, 3)


@pytest.mark.parametrize("seed,quant,zero_frac,trials", [(42, 8, 0.1, 60), (2024, 4, 0.05, 200)])
def test_csc_from_triplets_matches_oracle_exactly(seed, quant, zero_frac, trials):
    # test_sparse.py:59-70 and test_acceptance.py:273-285 (the dense left-to-right oracle)
    rng = np.random.default_rng(seed)
    for _ in range(trials):
        m = int(rng.integers(1, 51))
        n = int(rng.integers(1, 51))
        length = int(rng.integers(0, 501))
        i = rng.integers(0, m, length)
        j = rng.integers(0, n, length)
        k = np.round(rng.standard_normal(length) * quant) / quant
        k[rng.random(length) < zero_frac] = 0.0
        got = fa.csc_from_triplets(i, j, k, m, n)
        ref = fo.matlab_sparse(i, j, k, m, n)
        assert_same_csc((got.col_ptr, got.row_idx, got.values), ref)


def test_csc_from_triplets_long_runs_and_large_keys():
    rng = np.random.default_rng(1)
    i = np.concatenate([np.zeros(500, dtype=np.int64), rng.integers(0, 70000, 20000)])
    j = np.concatenate([np.zeros(500, dtype=np.int64), rng.integers(0, 90000, 20000)])
    v = rng.standard_normal(i.size)
    got = fa.csc_from_triplets(i, j, v, 70000, 90000)
    ref = fo.matlab_sparse(i, j, v, 70000, 90000)
    assert_same_csc((got.col_ptr, got.row_idx, got.values), ref)


@pytest.mark.parametrize("kind", list(fa.MatrixKind))
def test_assemble_all_strategies_match_reference(golden, kind):
    """OPTV2 is bitwise the reference's OPTV2; the element-loop strategies agree with it to
    roundoff (the reference's own contract, test_acceptance.py:87-106)."""
    name = "seeded_n16_s0"
    mesh = mesh_of(golden, name)
    kw = {}
    if kind is fa.MatrixKind.WEIGHTED_MASS:
        kw["weight"] = fa.WeightField.samples(golden[f"{name}/w"])
    if kind is fa.MatrixKind.ELASTIC:
        kw["params"] = fa.ElasticParams(*golden[f"{name}/elastic/lam_mu"])
    ref = tuple(golden[f"{name}/{kind.value}/{f}"] for f in ("col_ptr", "row_idx", "values"))
    m2 = fa.assemble(mesh, kind, fa.Strategy.OPTV2, **kw)
    assert_same_csc((m2.col_ptr, m2.row_idx, m2.values), ref, f"{kind}/OPTV2")
    scale = np.abs(m2.values).max()
    for strategy in (fa.Strategy.CLASSICAL, fa.Strategy.OPTV0, fa.Strategy.OPTV1):
        m = fa.assemble(mesh, kind, strategy, **kw)
        assert m.shape == (kind.n_dof(mesh.nq),) * 2
        assert fa.max_abs_diff(m, m2) <= 1e-12 * scale, f"{kind}/{strategy}"


@pytest.fixture(scope="module")
def loops():
    from conftest import GOLDEN

    d = np.load(GOLDEN / "loop_cases.npz")
    return {k: d[k] for k in d.files}


@pytest.mark.parametrize("strategy", ["CLASSICAL", "OPTV0", "OPTV1"])
@pytest.mark.parametrize("kind", ["mass", "massw", "stiff", "elastic"])
@pytest.mark.parametrize("name", ["square_n4", "disk_n4", "seeded_n5_s1"])
def test_element_loop_strategies_bitwise(loops, name, kind, strategy):
    """CLASSICAL / OPTV0 / OPTV1 bitwise against the reference's own element loops
    (assembly.py:359-397): per-element formulas (elements.py), CscBuilder's explicit zeros for
    CLASSICAL / OPTV0 (sparse.py:208-290), Matlab sparse() for OPTV1."""
    mesh = fa.Mesh(loops[f"{name}/V"], loops[f"{name}/C"])
    kw = {}
    if kind == "massw":
        kw["weight"] = fa.WeightField.quadratic()
    if kind == "elastic":
        kw["params"] = fa.ElasticParams(2.0, 0.7)
    m = fa.assemble(mesh, fa.MatrixKind(kind), getattr(fa.Strategy, strategy), **kw)
    ref = tuple(loops[f"{name}/{kind}/{strategy}/{f}"] for f in ("col_ptr", "row_idx", "values"))
    assert_same_csc((m.col_ptr, m.row_idx, m.values), ref, f"{name}/{kind}/{strategy}")


def test_incremental_keeps_zeros_triplet_drops_them():
    """test_assembly.py:269-276: on the unit square the stiffness has exact-zero sums; the
    CscBuilder strategies store them, the triplet strategies drop them."""
    mesh = fa.generate_unit_square_mesh(4)
    classical = fa.assemble(mesh, fa.MatrixKind.STIFFNESS, fa.Strategy.CLASSICAL)
    optv2 = fa.assemble(mesh, fa.MatrixKind.STIFFNESS, fa.Strategy.OPTV2)
    assert classical.nnz > optv2.nnz
    assert (classical.values == 0.0).any() and not (optv2.values == 0.0).any()
    assert fa.max_abs_diff(classical, optv2) <= 1e-14


def test_elem_functions_bitwise(loops):
    """elem_mass / elem_mass_weighted / elem_stiff / elem_stiff_elastic bitwise against the
    reference's per-element arithmetic (elements.py:34-154) on 64 random triangles."""
    P, A, W = loops["elem/P"], loops["elem/A"], loops["elem/W"]
    params = fa.ElasticParams(*loops["elem/lam_mu"])
    for t in range(len(A)):
        got = {
            "mass": fa.elem_mass(A[t]),
            "massw": fa.elem_mass_weighted(A[t], *W[t]),
            "stiff": fa.elem_stiff(P[t, 0], P[t, 1], P[t, 2], A[t]),
            "elastic": fa.elem_stiff_elastic(P[t, 0], P[t, 1], P[t, 2], A[t], params),
        }
        for k, g in got.items():
            ref = loops[f"elem/{k}"][t]
            assert np.array_equal(g.view(np.int64), ref.view(np.int64)), f"elem {k} triangle {t}"


def test_assemble_reference_invariants():
    # test_assembly.py:200-209, :247-259, :286-295 and acceptance criterion 3
    mesh = fa.generate_unit_square_mesh(8)
    m = fa.assemble(mesh, fa.MatrixKind.MASS, fa.Strategy.OPTV2)
    assert abs(m.values.sum() - 1.0) <= 1e-12
    s = fa.assemble(mesh, fa.MatrixKind.STIFFNESS, fa.Strategy.OPTV2)
    assert np.abs(s.to_dense() @ np.ones(mesh.nq)).max() <= 1e-10 * np.abs(s.values).max()
    k = fa.assemble(mesh, fa.MatrixKind.ELASTIC, fa.Strategy.OPTV2, params=fa.ElasticParams(1.0, 1.0)).to_dense()
    rot = np.zeros(2 * mesh.nq)
    rot[0::2] = -mesh.vertices[:, 1]
    rot[1::2] = mesh.vertices[:, 0]
    assert np.abs(k @ rot).max() <= 1e-9 * np.abs(k).max() * max(1.0, np.abs(rot).max())
    disk = fa.generate_disk_mesh(4)
    for kind, kw in ((fa.MatrixKind.MASS, {}), (fa.MatrixKind.STIFFNESS, {})):
        d = fa.assemble(disk, kind, fa.Strategy.OPTV2, **kw).to_dense()
        assert np.abs(d - d.T).max() == 0.0
    mw = fa.assemble(disk, fa.MatrixKind.WEIGHTED_MASS, fa.Strategy.OPTV2, weight=fa.WeightField.one())
    assert fa.max_abs_diff(fa.assemble(disk, fa.MatrixKind.MASS, fa.Strategy.OPTV2), mw) <= 1e-15


def test_budget_and_missing_parameters():
    mesh = fa.generate_unit_square_mesh(4)
    with pytest.raises(fa.AssemblyBudgetExceeded):
        fa.assemble(mesh, fa.MatrixKind.MASS, fa.Strategy.CLASSICAL, budget_s=0.0)
    fa.assemble(mesh, fa.MatrixKind.MASS, fa.Strategy.OPTV2, budget_s=0.0)  # OPTV2 ignores the budget
    with pytest.raises(ValueError, match="WeightField"):
        fa.assemble(mesh, fa.MatrixKind.WEIGHTED_MASS, fa.Strategy.OPTV2)


def test_paper_entry_points_and_handoff(golden):
    name = "seeded_n16_s1"
    V, C, w = golden[f"{name}/V"], golden[f"{name}/C"], golden[f"{name}/w"]
    areas = golden[f"{name}/areas"]
    nq, nme = V.shape[0], C.shape[0]
    cases = [
        ("mass", fa.MassAssemblingP1OptV2(nq, nme, C, areas)),
        ("massw", fa.MassWAssemblingP1OptV2(nq, nme, C, areas, w)),
        ("stiff", fa.StiffAssemblingP1OptV2(nq, nme, V, C, areas)),
        ("elastic", fa.StiffElasAssemblingP1OptV2(nq, nme, V, C, areas, 2.0, 0.7)),
    ]
    for kind, m in cases:
        ref = tuple(golden[f"{name}/{kind}/{f}"] for f in ("col_ptr", "row_idx", "values"))
        assert_same_csc((m.col_ptr, m.row_idx, m.values), ref, kind)
    mesh = fa.Mesh(V, C)
    m = fa.assemble(mesh, fa.MatrixKind.STIFFNESS, fa.Strategy.OPTV2)
    sp = m.to_scipy()
    assert np.array_equal(sp.toarray(), m.to_dense())
    t = m.to_torch_sparse_csr()
    assert np.array_equal(t.to_dense().cpu().numpy(), m.to_dense())
    # zero-copy hand-off: the CSR column ids are the device array itself
    assert t.col_indices().data_ptr() == m.device_arrays()[1].data_ptr()


def test_mesh_text_roundtrip_and_generators(golden, tmp_path):
    for name, mesh in (("square_n4", fa.generate_unit_square_mesh(4)), ("disk_n6", fa.generate_disk_mesh(6))):
        assert np.array_equal(mesh.vertices, golden[f"{name}/V"])
        assert np.array_equal(mesh.connectivity, golden[f"{name}/C"])
        p = tmp_path / f"{name}.msh"
        fa.write_mesh(mesh, p)
        assert fa.read_mesh(p) == mesh


@pytest.mark.parametrize("kind", ("massw", "stiff", "elastic"))
def test_host_assembler_pipelined_slots(golden, kind):
    """submit/result over two buffer slots: step i+1's copies and kernels are queued before
    step i is collected; every step must equal its own reference assembly."""
    import torch

    names = ["seeded_n16_s0", "seeded_n16_s1"] * 3
    V0, C0 = golden[f"{names[0]}/V"], golden[f"{names[0]}/C"]
    ha = fa.HostAssembler(kind, V0.shape[0], C0.shape[0], depth=2)
    pin = lambda x: torch.from_numpy(np.ascontiguousarray(x)).pin_memory()  # noqa: E731
    inputs = [(pin(golden[f"{n}/C"].astype(np.int32)), pin(golden[f"{n}/V"]), pin(golden[f"{n}/areas"]),
               pin(golden[f"{n}/w"]) if kind == "massw" else None) for n in names]
    tickets, got = [], []
    for i, (me, q, a, w) in enumerate(inputs):
        lam, mu = golden[f"{names[i]}/{kind}/lam_mu"]
        tickets.append(ha.submit(me, q if kind != "massw" else None, a, w, lam, mu))
        if i >= 1:
            rp, cc, vv, nnz = ha.result(tickets[i - 1])
            got.append((rp.numpy().copy(), cc.numpy().astype(np.int64), vv.numpy().copy()))
    rp, cc, vv, nnz = ha.result(tickets[-1])
    got.append((rp.numpy().copy(), cc.numpy().astype(np.int64), vv.numpy().copy()))
    for n, g in zip(names, got):
        ref = tuple(golden[f"{n}/{kind}/{f}"] for f in ("col_ptr", "row_idx", "values"))
        assert_same_csc(g, ref, n)
    with pytest.raises(ValueError, match="not in flight"):
        ha.result(tickets[-1])


@pytest.mark.parametrize("kind", ("mass", "massw", "stiff", "elastic"))
def test_paper_entry_point_rejects_out_of_range_ids(golden, kind):
    """An out-of-range vertex id raises ValueError (csc_from_triplets, sparse.py:131-137); the
    triangle is left out of the plan, so no kernel reads past q / w."""
    name = "seeded_n16_s0"
    V, C, w, areas = (golden[f"{name}/{f}"] for f in ("V", "C", "w", "areas"))
    nq, nme = V.shape[0], C.shape[0]
    bad = C.copy()
    bad[7, 1] = nq + 1000
    bad[9, 2] = -5
    call = {
        "mass": lambda c: fa.MassAssemblingP1OptV2(nq, nme, c, areas),
        "massw": lambda c: fa.MassWAssemblingP1OptV2(nq, nme, c, areas, w),
        "stiff": lambda c: fa.StiffAssemblingP1OptV2(nq, nme, V, c, areas),
        "elastic": lambda c: fa.StiffElasAssemblingP1OptV2(nq, nme, V, c, areas, *golden[f"{name}/elastic/lam_mu"]),
    }[kind]
    with pytest.raises(ValueError, match="out of range"):
        call(bad)
    m = call(C)  # the device is still healthy
    ref = tuple(golden[f"{name}/{kind}/{f}"] for f in ("col_ptr", "row_idx", "values"))
    assert_same_csc((m.col_ptr, m.row_idx, m.values), ref, kind)


def test_read_mesh_matches_reference_end_to_end(tmp_path):
    """read_mesh (native parser or reference rules, then the device Mesh ingestion) gives
    femasm.read_mesh's arrays or its exact MeshFormatError for every golden text case."""
    import json

    from conftest import GOLDEN

    cases = json.loads((GOLDEN / "mesh_text_cases.json").read_text())
    for name, case in cases.items():
        p = tmp_path / f"{name}.txt"
        p.write_bytes(case["text"].encode("ascii"))
        if case["ok"]:
            m = fa.read_mesh(p)
            assert np.array_equal(m.vertices, np.array(case["vertices"])), name
            assert np.array_equal(m.connectivity, np.array(case["connectivity"])), name
        else:
            with pytest.raises(fa.MeshFormatError) as ei:
                fa.read_mesh(p)
            assert ei.value.line_no == case["line_no"], name
            assert str(ei.value).replace(str(p), "<path>") == case["message"], name


def test_mesh_ingestion_errors_in_reference_order():
    """Mesh(V, C) validates on the device (fa_mesh_ingest) with mesh.py:87-113's messages and
    order: range before repeated ids before degenerate areas; areas bitwise compute_areas."""
    V = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0], [2.0, 0.0]])
    with pytest.raises(ValueError, match=r"connectivity index out of range \[0, nq\)"):
        fa.Mesh(V, np.array([[0, 1, 1], [0, 1, 4]]))  # repeated AND out of range: range wins
    with pytest.raises(ValueError, match="triangle with repeated vertex indices"):
        fa.Mesh(V, np.array([[0, 1, 2], [0, 3, 3]]))
    with pytest.raises(fa.DegenerateTriangleError) as ei:
        fa.Mesh(V, np.array([[0, 1, 2], [0, 1, 3], [0, 3, 1]]))
    assert ei.value.index == 1 and ei.value.area == 0.0
    with pytest.raises(ValueError, match=r"connectivity index out of range \[0, nq\)"):
        fa.Mesh(V, np.array([[0, 1, -1]]))
    from oracle import femasm_oracle as fo
    from paper_1305_3122_b200.meshgen import seeded_square_mesh

    sm = seeded_square_mesh(64, 2)
    m = fa.Mesh(sm.vertices, sm.connectivity)
    assert np.array_equal(m.areas.view(np.int64), fo.triangle_areas(sm.vertices, sm.connectivity).view(np.int64))
    me, q, a = m.device_arrays()
    assert np.array_equal(me.cpu().numpy(), sm.connectivity.astype(np.int32))
