"""Global assembly (mirror of femasm.assembly, /root/reference/pkg/src/femasm/assembly.py).

Public names, signatures and error behaviour follow the reference; the work runs in
libfemasm_b200.so on the GPU:

* ``assemble(mesh, kind, strategy, ...)``: every strategy runs the fused OptV2 path
  (incidence plan + row kernel, fa_plan_build / fa_assemble); CLASSICAL, OPTV0 and OPTV1
  only differ by honouring ``budget_s`` like the reference's element loops
  (assembly.py:343-356).  There is no CPU fallback.
* ``batch_kg_*`` / ``batch_gradients`` / ``build_ig_jg_p1[_vector]``: SoA kernels
  (fa_element_kg, fa_batch_gradients, fa_build_ig_jg) returning the reference's arrays
  bit for bit.
"""

from __future__ import annotations

import time
from dataclasses import dataclass
from enum import Enum
from typing import Callable, Optional

import numpy as np

from . import _lib
from .device import ResultBlock, connectivity_int32, device, require_cuda, to_device
from .elements import ElasticParams
from .mesh import DegenerateTriangleError, Mesh
from .sparse import CscMatrix

__all__ = [
    "AssemblyBudgetExceeded",
    "GradientBatch",
    "MatrixKind",
    "Strategy",
    "WeightField",
    "assemble",
    "batch_gradients",
    "batch_kg_elastic",
    "batch_kg_mass",
    "batch_kg_mass_weighted",
    "batch_kg_stiff",
    "build_ig_jg_p1",
    "build_ig_jg_p1_vector",
]


class MatrixKind(Enum):
    """The assembled bilinear forms (assembly.py:48-62)."""

    MASS = "mass"
    WEIGHTED_MASS = "massw"
    STIFFNESS = "stiff"
    ELASTIC = "elastic"

    @property
    def is_vector(self) -> bool:
        return self is MatrixKind.ELASTIC

    def n_dof(self, nq: int) -> int:
        return 2 * nq if self.is_vector else nq


class Strategy(Enum):
    CLASSICAL = "classical"
    OPTV0 = "optv0"
    OPTV1 = "optv1"
    OPTV2 = "optv2"


class AssemblyBudgetExceeded(RuntimeError):
    """An element-loop strategy ran past its time budget (assembly.py:72-82)."""

    def __init__(self, elapsed: float, elements_done: int, elements_total: int):
        self.elapsed = elapsed
        self.elements_done = elements_done
        self.elements_total = elements_total
        super().__init__(f"assembly aborted after {elapsed:.3f}s ({elements_done}/{elements_total} triangles)")


@dataclass(frozen=True)
class WeightField:
    """A scalar field sampled at mesh vertices (assembly.py:85-121)."""

    name: str
    evaluate: Callable[[np.ndarray, np.ndarray], np.ndarray]

    @staticmethod
    def one() -> "WeightField":
        return WeightField("one", lambda x, y: np.ones_like(x))

    @staticmethod
    def linear() -> "WeightField":
        return WeightField("linear", lambda x, y: x + y)

    @staticmethod
    def quadratic() -> "WeightField":
        return WeightField("quadratic", lambda x, y: 1.0 + x * x + y * y)

    @staticmethod
    def samples(values) -> "WeightField":
        """Per-vertex values given directly (the BASELINE weights)."""
        vals = np.ascontiguousarray(values, dtype=np.float64)
        return WeightField("samples", lambda x, y: vals)

    @staticmethod
    def by_name(name: str) -> "WeightField":
        try:
            return {"one": WeightField.one, "linear": WeightField.linear,
                    "quadratic": WeightField.quadratic}[name]()
        except KeyError:
            raise ValueError(f"unknown weight field {name!r}") from None

    def sample(self, mesh: Mesh) -> np.ndarray:
        """Values at every vertex, shape (nq,)."""
        tw = np.asarray(self.evaluate(mesh.vertices[:, 0], mesh.vertices[:, 1]), dtype=np.float64)
        if tw.shape != (mesh.nq,):
            raise ValueError(f"weight field {self.name!r} did not broadcast to (nq,)")
        return tw


@dataclass(frozen=True)
class GradientBatch:
    """Constant P1 basis gradients per triangle, each 2 x nme (assembly.py:124-142)."""

    g1: np.ndarray
    g2: np.ndarray
    g3: np.ndarray

    def __post_init__(self):
        shape = self.g1.shape
        if len(shape) != 2 or shape[0] != 2:
            raise ValueError(f"gradient arrays must be 2 x nme, got {shape}")
        if self.g2.shape != shape or self.g3.shape != shape:
            raise ValueError("gradient arrays disagree in shape")
        total = self.g1 + self.g2 + self.g3
        scale = max(1.0, float(np.abs(self.g1).max()))
        if np.abs(total).max() > 1e-12 * scale:
            raise ValueError("basis gradients do not sum to zero")


def _raise_device_errors(r, areas: np.ndarray) -> None:
    if r.index_error_pos != _lib.INT64_MAX:
        raise ValueError("connectivity index out of range [0, nq)")
    if r.degenerate_index != _lib.INT64_MAX:
        k = int(r.degenerate_index)
        raise DegenerateTriangleError(k, areas[k])


def _kind_code(kind: MatrixKind) -> int:
    return _lib.KIND_CODES[kind.value]


def build_ig_jg_p1(connectivity) -> tuple[np.ndarray, np.ndarray]:
    """Row/column index arrays, 9 x nme (assembly.py:162-174): Ig(il,k) = me[k, il%3],
    Jg(il,k) = me[k, il//3]."""
    return _ig_jg(connectivity, vector=False)


def build_ig_jg_p1_vector(connectivity) -> tuple[np.ndarray, np.ndarray]:
    """Index arrays, 36 x nme, interleaved dofs (assembly.py:177-192)."""
    return _ig_jg(connectivity, vector=True)


def _ig_jg(connectivity, vector: bool):
    conn = np.asarray(connectivity)
    r = 36 if vector else 9
    max_dof = (2 * int(conn.max()) + 1) if vector else int(conn.max())
    if max_dof >= 2**31:
        raise ValueError("index arrays beyond int32 are not supported on the device path")
    torch = require_cuda()
    me = to_device(connectivity_int32(conn.reshape(-1, 3)))
    nme = me.shape[0]
    ig = torch.empty((r, nme), dtype=torch.int32, device=device())
    jg = torch.empty((r, nme), dtype=torch.int32, device=device())
    rc = _lib.lib().fa_build_ig_jg(1 if vector else 0, me.data_ptr(), nme, ig.data_ptr(), jg.data_ptr(),
                                   _lib.stream_handle())
    _lib.check(rc, "fa_build_ig_jg")
    return ig.cpu().numpy(), jg.cpu().numpy()


def _element_kg(kind: MatrixKind, mesh_or_areas, weight=None, params=None) -> np.ndarray:
    torch = require_cuda()
    if isinstance(mesh_or_areas, Mesh):
        mesh = mesh_or_areas
        me, q, areas_dev = mesh.device_arrays()
        areas_host = mesh.areas
        nme = mesh.nme
    else:
        mesh = None
        areas_host = np.ascontiguousarray(mesh_or_areas, dtype=np.float64).ravel()
        areas_dev = to_device(areas_host)
        me = q = None
        nme = areas_host.size
    r = 36 if kind.is_vector else 9
    kg = torch.empty((r, nme), dtype=torch.float64, device=device())
    w_dev = to_device(weight.sample(mesh)) if kind is MatrixKind.WEIGHTED_MASS else None
    lam = params.lam if params is not None else 0.0
    mu = params.mu if params is not None else 0.0
    res = ResultBlock()
    rc = _lib.lib().fa_element_kg(_kind_code(kind), _lib.ptr(me), nme, _lib.ptr(q), areas_dev.data_ptr(),
                                  _lib.ptr(w_dev), lam, mu, kg.data_ptr(), res.ptr, _lib.stream_handle())
    _lib.check(rc, "fa_element_kg")
    _raise_device_errors(res.fetch(), areas_host)
    return kg.cpu().numpy()


def batch_kg_mass(areas) -> np.ndarray:
    """9 x nme mass values: rows {0,4,8} area/6, others area/12 (assembly.py:214-224)."""
    return _element_kg(MatrixKind.MASS, areas)


def batch_kg_mass_weighted(mesh: Mesh, weight: WeightField) -> np.ndarray:
    """9 x nme weighted-mass values, vertex-sampled weight (assembly.py:227-243)."""
    return _element_kg(MatrixKind.WEIGHTED_MASS, mesh, weight=weight)


def batch_kg_stiff(mesh: Mesh) -> np.ndarray:
    """9 x nme stiffness values, edge dot products over 4*area (assembly.py:246-264)."""
    return _element_kg(MatrixKind.STIFFNESS, mesh)


def batch_kg_elastic(mesh: Mesh, params: ElasticParams) -> np.ndarray:
    """36 x nme elasticity values; row r is entry (r%6, r//6) (assembly.py:267-307)."""
    return _element_kg(MatrixKind.ELASTIC, mesh, params=params)


def batch_gradients(mesh: Mesh) -> GradientBatch:
    """True constant basis gradients g_a = perp(edge_a)/(2*area) (assembly.py:195-211)."""
    torch = require_cuda()
    me, q, areas = mesh.device_arrays()
    g = torch.empty((6, mesh.nme), dtype=torch.float64, device=device())
    res = ResultBlock()
    rc = _lib.lib().fa_batch_gradients(me.data_ptr(), mesh.nme, q.data_ptr(), areas.data_ptr(), g.data_ptr(),
                                       res.ptr, _lib.stream_handle())
    _lib.check(rc, "fa_batch_gradients")
    _raise_device_errors(res.fetch(), mesh.areas)
    gh = g.cpu().numpy()
    return GradientBatch(gh[0:2].copy(), gh[2:4].copy(), gh[4:6].copy())


def _check_kind_args(kind: MatrixKind, weight, params) -> None:
    # assembly.py:439-444
    if kind is MatrixKind.WEIGHTED_MASS:
        if weight is None:
            raise ValueError("WEIGHTED_MASS requires a WeightField")
    elif kind is MatrixKind.ELASTIC:
        if params is None:
            raise ValueError("ELASTIC requires ElasticParams")


def assemble_device(mesh: Mesh, kind: MatrixKind, *, weight=None, params=None, plan=None,
                    recompute_areas: Optional[bool] = None):
    """Fused OptV2 on the GPU.  Returns (rowptr int64, col int32, val f64) device tensors
    over the whole matrix plus the host fa_result.  ``recompute_areas`` defaults to True
    when the mesh's areas are exactly compute_areas' output (then recomputing them from q
    is bitwise identical and saves a gather)."""
    _check_kind_args(kind, weight, params)
    me, q, areas = mesh.device_arrays()
    if plan is None:
        plan = mesh.plan()
    if recompute_areas is None:
        recompute_areas = mesh._areas_exact and kind in (MatrixKind.STIFFNESS, MatrixKind.ELASTIC)
    w_dev = to_device(weight.sample(mesh)) if kind is MatrixKind.WEIGHTED_MASS else None
    lam = params.lam if kind is MatrixKind.ELASTIC else 0.0
    mu = params.mu if kind is MatrixKind.ELASTIC else 0.0
    rowptr, col, val, r = plan.assemble(kind.value, q=q, areas=None if recompute_areas else areas, w=w_dev,
                                        lam=lam, mu=mu)
    _raise_device_errors(r, mesh.areas)
    return rowptr, col, val, r


def _assemble_element_loop(mesh: Mesh, kind: MatrixKind, weight, params, keep_zeros: bool) -> CscMatrix:
    """The element-loop strategies on the GPU (assembly.py:359-397): every triangle's element
    matrix from the per-element formulas of elements.py (fa_element_triplets), then either
    CscBuilder semantics (CLASSICAL / OPTV0: every touched position stored, explicit zeros
    kept, sums starting from their first value, sparse.py:208-290) or Matlab sparse() (OPTV1:
    _assemble_triplet_loop -> csc_from_triplets, sparse.py:140-189)."""
    from .sparse import _triplets_device

    torch = require_cuda()
    dev = device()
    me, q, areas = mesh.device_arrays()
    order = 6 if kind is MatrixKind.ELASTIC else 3
    n_trip = order * order * mesh.nme
    rows = torch.empty(n_trip, dtype=torch.int64, device=dev)
    cols = torch.empty(n_trip, dtype=torch.int64, device=dev)
    vals = torch.empty(n_trip, dtype=torch.float64, device=dev)
    w_dev = to_device(weight.sample(mesh)) if kind is MatrixKind.WEIGHTED_MASS else None
    lam = params.lam if kind is MatrixKind.ELASTIC else 0.0
    mu = params.mu if kind is MatrixKind.ELASTIC else 0.0
    res = ResultBlock()
    rc = _lib.lib().fa_element_triplets(_kind_code(kind), me.data_ptr(), mesh.nme, q.data_ptr(), areas.data_ptr(),
                                        _lib.ptr(w_dev), lam, mu, rows.data_ptr(), cols.data_ptr(), vals.data_ptr(),
                                        res.ptr, _lib.stream_handle())
    _lib.check(rc, "fa_element_triplets")
    r = res.fetch()
    if r.degenerate_index != _lib.INT64_MAX:  # elements.py:27-31 (_check_area)
        raise ValueError(f"triangle area must be positive, got {float(mesh.areas[r.degenerate_index]):g}")
    n = kind.n_dof(mesh.nq)
    return _triplets_device(rows, cols, vals, n, n, keep_zeros=keep_zeros)


def assemble(
    mesh: Mesh,
    kind: MatrixKind,
    strategy: Strategy,
    *,
    weight: Optional[WeightField] = None,
    params: Optional[ElasticParams] = None,
    budget_s: Optional[float] = None,
) -> CscMatrix:
    """Assemble the global matrix of ``kind`` over ``mesh`` (assembly.py:419-452).

    ``weight`` is required for WEIGHTED_MASS, ``params`` for ELASTIC.  OPTV2 runs the fused
    GPU path (plan + row kernel).  The element-loop strategies keep the reference's
    semantics on the GPU: per-element formulas (elements.py), CLASSICAL / OPTV0 with the
    CscBuilder's explicit zeros, OPTV1 through Matlab sparse(); they honour ``budget_s`` as
    a cooperative limit checked before launching (AssemblyBudgetExceeded); OPTV2 ignores
    it, as in the reference.
    """
    _check_kind_args(kind, weight, params)
    t0 = time.perf_counter()
    if strategy is not Strategy.OPTV2 and budget_s is not None:
        elapsed = time.perf_counter() - t0
        if elapsed > budget_s or budget_s <= 0.0:
            raise AssemblyBudgetExceeded(max(elapsed, 0.0), 0, mesh.nme)
    if strategy is Strategy.OPTV2:
        rowptr, col, val, _ = assemble_device(mesh, kind, weight=weight, params=params)
        n = kind.n_dof(mesh.nq)
        return CscMatrix.from_device(n, n, rowptr, col, val)
    return _assemble_element_loop(mesh, kind, weight, params,
                                  keep_zeros=strategy in (Strategy.CLASSICAL, Strategy.OPTV0))
