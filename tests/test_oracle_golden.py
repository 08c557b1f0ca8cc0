"""Pin the CPU oracle (numpy restatement + C restatement) against the real reference.

The fixtures were produced by tests/golden/make_golden.py running femasm itself; these
tests need no GPU and run in the CPU suite.
"""

import numpy as np
import pytest

from helpers import assert_same_csc, csc_digests, mesh_digest
from oracle import c_oracle
from oracle import femasm_oracle as fo
from paper_1305_3122_b200.meshgen import BASELINE_CONFIGS, seeded_square_mesh

KINDS = ("mass", "massw", "stiff", "elastic")
SEEDED = [f"seeded_n{n}_s{s}" for n in (2, 5, 16) for s in (0, 1)]


def _case(golden, name):
    V, C = golden[f"{name}/V"], golden[f"{name}/C"]
    w = golden.get(f"{name}/w")
    if w is None:
        w = 1.0 + V[:, 0] ** 2 + V[:, 1] ** 2  # WeightField.quadratic (assembly.py:100-103)
    return V, C, w


def _params(golden, name, kind):
    lm = golden.get(f"{name}/{kind}/lam_mu")
    if lm is not None:
        return float(lm[0]), float(lm[1])
    return 1.0, 1.0


@pytest.mark.parametrize("name", SEEDED + ["square_n4", "square_n1", "disk_n4", "disk_n6"])
def test_areas_match_reference(golden, name):
    V, C, _ = _case(golden, name)
    ref = golden[f"{name}/areas"]
    assert np.array_equal(fo.triangle_areas(V, C), ref)
    assert np.array_equal(c_oracle.areas(V, C), ref)


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("name", SEEDED + ["square_n4", "square_n1", "disk_n4", "disk_n6"])
def test_numpy_oracle_matches_reference(golden, name, kind):
    V, C, w = _case(golden, name)
    lam, mu = _params(golden, name, kind)
    got = fo.assemble_optv2(kind, V, C, golden[f"{name}/areas"], w, lam, mu)
    ref = tuple(golden[f"{name}/{kind}/{f}"] for f in ("col_ptr", "row_idx", "values"))
    assert_same_csc(got, ref, f"{name}/{kind}")


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("name", SEEDED + ["square_n4", "disk_n6"])
def test_c_oracle_matches_reference(golden, name, kind):
    V, C, w = _case(golden, name)
    lam, mu = _params(golden, name, kind)
    got = c_oracle.assemble(kind, V, C, golden[f"{name}/areas"], w, lam, mu)
    ref = tuple(golden[f"{name}/{kind}/{f}"] for f in ("col_ptr", "row_idx", "values"))
    assert_same_csc(got, ref, f"{name}/{kind}")


@pytest.mark.parametrize("name", SEEDED)
def test_element_values_match_reference(golden, name):
    V, C, w = _case(golden, name)
    areas = golden[f"{name}/areas"]
    for kind, key in (("mass", "kg_mass"), ("massw", "kg_massw"), ("stiff", "kg_stiff"), ("elastic", "kg_elastic")):
        ref = golden[f"{name}/{key}"]
        for got in (fo.element_values(kind, V, C, areas, w, 1.0, 0.5),
                    c_oracle.element_values(kind, V, C, areas, w, 1.0, 0.5)):
            assert np.array_equal(got.view(np.int64), ref.view(np.int64)), (name, kind)


def test_generator_matches_reference_meshes(digests):
    """The seeded generator is pinned: the digests were computed from the arrays the
    reference assembled."""
    for key, d in digests.items():
        if d["N"] > 1024:
            continue
        sm = seeded_square_mesh(d["N"], d["seed"])
        assert mesh_digest(sm) == d["mesh_sha256"], key


@pytest.mark.parametrize("key", ["C1/s0", "C1/s1", "C1/s2", "EL64/s0"])
def test_numpy_oracle_matches_reference_digest(digests, key):
    d = digests[key]
    sm = seeded_square_mesh(d["N"], d["seed"])
    areas = fo.triangle_areas(sm.vertices, sm.connectivity)
    out = fo.assemble_optv2(d["kind"], sm.vertices, sm.connectivity, areas, sm.weights, d["lam"], d["mu"])
    assert len(out[2]) == d["nnz"]
    assert csc_digests(*out) == (d["col_ptr_sha256"], d["row_idx_sha256"], d["values_sha256"])


@pytest.mark.parametrize("key", ["C1/s0", "EL64/s0", "C2/s0"])
def test_c_oracle_matches_reference_digest(digests, key):
    if key not in digests:
        pytest.skip(f"{key} digest not generated")
    d = digests[key]
    sm = seeded_square_mesh(d["N"], d["seed"])
    areas = c_oracle.areas(sm.vertices, sm.connectivity)
    out = c_oracle.assemble(d["kind"], sm.vertices, sm.connectivity, areas, sm.weights, d["lam"], d["mu"])
    assert len(out[2]) == d["nnz"]
    assert csc_digests(*out) == (d["col_ptr_sha256"], d["row_idx_sha256"], d["values_sha256"])


def test_row_block_subset_oracle_is_exact(golden):
    """assembling only the triangles touching a row block reproduces the
    block of the full assembly bit for bit (basis of the multi-GPU parity tests)."""
    name = "seeded_n16_s0"
    V, C, w = _case(golden, name)
    areas = golden[f"{name}/areas"]
    for kind in KINDS:
        full = fo.assemble_optv2(kind, V, C, areas, w, 1.0, 0.5)
        rpv = 2 if kind == "elastic" else 1
        nq = V.shape[0]
        cuts = np.linspace(0, nq, 5).astype(int)
        for v0, v1 in zip(cuts[:-1], cuts[1:]):
            ptr, idx, vals = fo.assemble_row_block(kind, V, C, areas, w, 1.0, 0.5, v0, v1)
            lo, hi = full[0][rpv * v0], full[0][rpv * v1]
            assert np.array_equal(ptr, full[0][rpv * v0: rpv * v1 + 1] - lo)
            assert np.array_equal(idx, full[1][lo:hi])
            assert np.array_equal(vals, full[2][lo:hi])
            cp = c_oracle.assemble(kind, V, C, areas, w, 1.0, 0.5, rpv * v0, rpv * v1)
            assert np.array_equal(cp[0], ptr) and np.array_equal(cp[1], idx) and np.array_equal(cp[2], vals)


def test_matlab_sparse_reference_examples():
    """Worked example and edge cases of the reference tests (test_sparse.py:16-47)."""
    p, i, v = fo.matlab_sparse([0, 1, 2, 2, 0, 1], [0, 1, 1, 2, 3, 3], [1.0, 5.0, 1.0, 2.0, 6.0, 4.0], 3, 4)
    assert v.tolist() == [1, 5, 1, 2, 6, 4] and i.tolist() == [0, 1, 2, 2, 0, 1] and p.tolist() == [0, 1, 3, 4, 6]
    p, i, v = fo.matlab_sparse([0, 0], [0, 0], [2.0, 3.0], 1, 1)
    assert v.tolist() == [5.0]
    p, i, v = fo.matlab_sparse([0, 0], [0, 0], [2.0, -2.0], 1, 1)
    assert v.size == 0 and p.tolist() == [0, 0]
    p, i, v = fo.matlab_sparse([0, 1], [0, 0], [0.0, 1.0], 2, 1)
    assert i.tolist() == [1] and v.tolist() == [1.0]
    p, i, v = fo.matlab_sparse([], [], [], 3, 3)
    assert v.size == 0 and p.tolist() == [0, 0, 0, 0]


def test_baseline_config_table():
    assert BASELINE_CONFIGS["C2"] == ("massw", 1024, None, None)
    assert BASELINE_CONFIGS["C4"][2:] == (1.0, 0.5)
