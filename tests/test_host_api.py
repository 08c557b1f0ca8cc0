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
