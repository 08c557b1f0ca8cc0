"""Host-side logic of the drop-in API (no GPU): types, validation, error messages, and the
no-CPU-fallback rule."""

import numpy as np
import pytest
import torch

import paper_1305_3122_b200 as fa
from paper_1305_3122_b200.assembly import _check_kind_args


def test_matrix_kind_dofs():
    assert fa.MatrixKind.MASS.n_dof(10) == 10
    assert fa.MatrixKind.ELASTIC.n_dof(10) == 20
    assert fa.MatrixKind.ELASTIC.is_vector and not fa.MatrixKind.STIFFNESS.is_vector
    assert [s.value for s in fa.Strategy] == ["classical", "optv0", "optv1", "optv2"]


def test_missing_parameters_messages():
    # assembly.py:439-444 / test_assembly.py:240-245
    with pytest.raises(ValueError, match="WeightField"):
        _check_kind_args(fa.MatrixKind.WEIGHTED_MASS, None, None)
    with pytest.raises(ValueError, match="ElasticParams"):
        _check_kind_args(fa.MatrixKind.ELASTIC, None, None)


def test_elastic_params_validation():
    p = fa.ElasticParams(1.0, 0.5)
    assert p.C[0, 0] == 2.0 and p.C[2, 2] == 0.5
    with pytest.raises(ValueError):
        fa.ElasticParams(-1.0, 0.5)
    with pytest.raises(ValueError):
        fa.ElasticParams(1.0, 0.0)
    assert fa.elasticity_tensor(2.0, 0.7) == fa.ElasticParams(2.0, 0.7)


def test_weight_field_names():
    assert fa.WeightField.by_name("quadratic").name == "quadratic"
    with pytest.raises(ValueError):
        fa.WeightField.by_name("nope")


def test_triplet_batch_shape_validation():
    ig = np.zeros((9, 2), dtype=np.int64)
    fa.TripletBatch(9, ig, ig, ig.astype(float))
    with pytest.raises(ValueError):
        fa.TripletBatch(8, ig[:8], ig[:8], ig[:8].astype(float))
    with pytest.raises(ValueError):
        fa.TripletBatch(9, ig, ig[:, :1], ig.astype(float))
    flat = fa.TripletBatch(9, np.arange(18).reshape(9, 2), np.arange(18).reshape(9, 2),
                           np.arange(18.0).reshape(9, 2)).flat()[0]
    assert flat[:9].tolist() == list(range(0, 18, 2))


def test_csc_matrix_host_semantics():
    # the worked example of test_sparse.py:16-31
    a = fa.CscMatrix(3, 4, [0, 1, 3, 4, 6], [0, 1, 2, 2, 0, 1], [1.0, 5.0, 1.0, 2.0, 6.0, 4.0])
    assert a.get(0, 3) == 6.0 and a.get(2, 3) == 0.0
    assert np.array_equal(a.to_dense(), [[1, 0, 0, 6], [0, 5, 0, 4], [0, 1, 2, 0]])
    with pytest.raises(ValueError):
        a.get(3, 0)
    with pytest.raises(AttributeError):
        a.n_rows = 5
    with pytest.raises(ValueError):
        fa.CscMatrix(3, 2, [0, 2, 1], [0, 1], [1.0, 2.0])
    with pytest.raises(ValueError, match="increase"):
        fa.CscMatrix(3, 1, [0, 2], [1, 0], [1.0, 2.0])
    big = fa.CscMatrix(100_000, 10_000, np.zeros(10_001, dtype=np.int64), [], [])
    with pytest.raises(ValueError, match="guard"):
        big.to_dense()


def test_matrix_market_writer(tmp_path):
    a = fa.CscMatrix(3, 4, [0, 1, 3, 4, 6], [0, 1, 2, 2, 0, 1], [1.0, 5.0, 1.0, 2.0, 6.0, 4.0])
    p = tmp_path / "a.mtx"
    fa.write_matrix_market(a, p)
    lines = p.read_text().splitlines()
    assert lines[0] == "%%MatrixMarket matrix coordinate real general"
    assert lines[1] == "3 4 6"
    import scipy.io

    assert np.array_equal(scipy.io.mmread(p).toarray(), a.to_dense())


def _reference_mtx(matrix, path):
    """femasm's writer, restated from sparse.py:332-339 (per-entry Python loop)."""
    rows, cols, vals = matrix.triplets()
    with open(path, "w", encoding="ascii") as f:
        f.write("%%MatrixMarket matrix coordinate real general\n")
        f.write(f"{matrix.n_rows} {matrix.n_cols} {matrix.nnz}\n")
        for i, j, v in zip(rows, cols, vals):
            f.write(f"{i + 1} {j + 1} {'%.17g' % v}\n")


@pytest.mark.parametrize("threads", (1, 3, 0))
def test_matrix_market_writer_is_byte_identical(tmp_path, threads):
    rng = np.random.default_rng(7)
    n_rows, n_cols = 500, 300
    dense = np.zeros((n_rows, n_cols))
    mask = rng.random((n_rows, n_cols)) < 0.05
    vals = rng.standard_normal(mask.sum()) * 10.0 ** rng.integers(-320, 300, mask.sum())
    special = np.array([1.0, -0.0, 0.1, 1e-5, 123456789.0, 2.0 ** -1074, 1.7976931348623157e308, -2.5])
    vals[: special.size] = special
    dense[mask] = vals
    dense[:, 17] = 0.0  # empty columns inside and at the end
    dense[:, -1] = 0.0
    nz = dense != 0.0
    nz[mask] = True
    nz[:, 17] = False
    nz[:, -1] = False
    cols = np.nonzero(nz.T)
    col_ptr = np.concatenate([[0], np.cumsum(nz.sum(axis=0))])
    a = fa.CscMatrix(n_rows, n_cols, col_ptr, cols[1], dense.T[nz.T])
    ours, ref = tmp_path / "ours.mtx", tmp_path / "ref.mtx"
    fa.write_matrix_market(a, ours, threads=threads)
    _reference_mtx(a, ref)
    assert ours.read_bytes() == ref.read_bytes()
    empty = fa.CscMatrix(4, 3, np.zeros(4, dtype=np.int64), [], [])
    fa.write_matrix_market(empty, ours, threads=threads)
    _reference_mtx(empty, ref)
    assert ours.read_bytes() == ref.read_bytes()


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback_without_gpu():
    with pytest.raises(RuntimeError, match="CUDA"):
        fa.compute_areas(np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0]]), np.array([[0, 1, 2]]))
    with pytest.raises(RuntimeError, match="CUDA"):
        fa.csc_from_triplets([0], [0], [1.0], 1, 1)
    with pytest.raises(RuntimeError, match="CUDA"):
        fa.batch_kg_mass(np.array([0.5]))


def test_product_package_never_imports_the_oracle():
    import pathlib

    pkg = pathlib.Path(fa.__file__).parent
    for f in pkg.rglob("*.py"):
        text = f.read_text()
        assert "import oracle" not in text and "from oracle" not in text, f


def _mesh_text_cases():
    import json

    from conftest import GOLDEN

    return json.loads((GOLDEN / "mesh_text_cases.json").read_text())


def test_mesh_text_parsers_match_reference(tmp_path):
    """read_mesh's two parsers against femasm.read_mesh's own results (tests/golden/
    mesh_text_cases.json, make_golden.py mesh_text): the native multithreaded one accepts the
    well-formed layout and defers everything else; the reference-equivalent one returns the
    same arrays or raises the same MeshFormatError (line number and text)."""
    from paper_1305_3122_b200 import mesh as M

    for name, case in _mesh_text_cases().items():
        p = tmp_path / f"{name}.txt"
        p.write_bytes(case["text"].encode("ascii"))
        native = M._read_mesh_native(p)
        mesh_error = not case["ok"] and "invalid mesh:" in case["message"]
        if case["ok"] or mesh_error:
            V, C = M._parse_mesh_text(p)
            if case["ok"]:
                assert np.array_equal(V, np.array(case["vertices"])), name
                assert np.array_equal(C, np.array(case["connectivity"])), name
            if native is not None:
                assert np.array_equal(native[0], V) and np.array_equal(native[1], C), name
            else:
                assert name == "python_tokens", f"{name}: well-formed file rejected by the native parser"
        else:
            assert native is None, name
            with pytest.raises(M.MeshFormatError) as ei:
                M._parse_mesh_text(p)
            assert ei.value.line_no == case["line_no"], name
            assert str(ei.value).replace(str(p), "<path>") == case["message"], name


def test_native_mesh_reader_large_file(tmp_path):
    """A seeded mesh written with write_mesh's format parses natively to the same arrays."""
    from paper_1305_3122_b200 import mesh as M
    from paper_1305_3122_b200.meshgen import seeded_square_mesh

    sm = seeded_square_mesh(120, 3)
    p = tmp_path / "m.txt"
    with open(p, "w") as f:
        f.write(f"{sm.nq} {sm.nme}\n")
        for x, y in sm.vertices:
            f.write("%.17g %.17g\n" % (x, y))
        for a, b, c in sm.connectivity:
            f.write(f"{a + 1} {b + 1} {c + 1}\n")
    V, C = M._read_mesh_native(p)
    assert np.array_equal(V, sm.vertices) and np.array_equal(C, sm.connectivity)
