"""Element-level API (mirror of femasm.elements, /root/reference/pkg/src/femasm/elements.py).

``ElasticParams`` / ``elasticity_tensor`` are the parameter types of the OptV2 elastic
path (elements.py:81-108) and are kept exactly.  The per-element matrices ``elem_*`` only
feed the reference's element-loop strategies, which are out of the B200 scope; they are
provided for API completeness and evaluate one triangle through the same GPU element
kernel as the batch path (fa_element_kg with nme = 1), so their values are bitwise those
of the batch kernels.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "ElasticParams",
    "elasticity_tensor",
    "elem_mass",
    "elem_mass_weighted",
    "elem_stiff",
    "elem_stiff_elastic",
]

AREA_EPS = 1e-300


@dataclass(frozen=True)
class ElasticParams:
    """Lame coefficients and the isotropic Hooke matrix C (elements.py:81-103).
    Admissibility: lam + mu > 0 and mu > 0."""

    lam: float
    mu: float
    C: np.ndarray = field(init=False, repr=False, compare=False)

    def __post_init__(self):
        lam, mu = float(self.lam), float(self.mu)
        if not lam + mu > 0.0:
            raise ValueError(f"lam + mu must be positive, got {lam + mu:g}")
        if not mu > 0.0:
            raise ValueError(f"mu must be positive, got {mu:g}")
        C = np.array([[lam + 2 * mu, lam, 0.0], [lam, lam + 2 * mu, 0.0], [0.0, 0.0, mu]])
        C.flags.writeable = False
        object.__setattr__(self, "lam", lam)
        object.__setattr__(self, "mu", mu)
        object.__setattr__(self, "C", C)


def elasticity_tensor(lam: float, mu: float) -> ElasticParams:
    return ElasticParams(lam, mu)


def _check_area(area: float) -> float:
    area = float(area)
    if not area > AREA_EPS:
        raise ValueError(f"triangle area must be positive, got {area:g}")
    return area


def _one_triangle(kind_code: int, pts, area: float, w=None, lam=0.0, mu=0.0) -> np.ndarray:
    """One element matrix with the per-element formulas of elements.py (fa_element_triplets:
    the arithmetic of the element-loop strategies, not the batch kernels')."""
    import torch

    from . import _lib
    from .device import ResultBlock, device, require_cuda

    require_cuda()
    dev = device()
    q = torch.tensor(np.asarray(pts, dtype=np.float64).reshape(3, 2), device=dev)
    me = torch.tensor([[0, 1, 2]], dtype=torch.int32, device=dev)
    areas = torch.tensor([area], dtype=torch.float64, device=dev)
    wd = torch.tensor(np.asarray(w, dtype=np.float64), device=dev) if w is not None else None
    order = 6 if kind_code == 3 else 3
    rows = torch.empty(order * order, dtype=torch.int64, device=dev)
    cols = torch.empty_like(rows)
    vals = torch.empty(order * order, dtype=torch.float64, device=dev)
    res = ResultBlock()
    rc = _lib.lib().fa_element_triplets(kind_code, me.data_ptr(), 1, q.data_ptr(), areas.data_ptr(), _lib.ptr(wd),
                                        float(lam), float(mu), rows.data_ptr(), cols.data_ptr(), vals.data_ptr(),
                                        res.ptr, _lib.stream_handle())
    _lib.check(rc, "fa_element_triplets")
    return vals.cpu().numpy().reshape(order, order, order="F").copy()


def elem_mass(area: float) -> np.ndarray:
    """(area/12) * [[2,1,1],[1,2,1],[1,1,2]] (elements.py:34-39)."""
    area = _check_area(area)
    return _one_triangle(0, np.zeros((3, 2)), area)


def elem_mass_weighted(area: float, w1: float, w2: float, w3: float) -> np.ndarray:
    """Vertex-sampled weighted mass matrix (elements.py:42-57)."""
    area = _check_area(area)
    return _one_triangle(1, np.zeros((3, 2)), area, w=[w1, w2, w3])


def elem_stiff(p1, p2, p3, area: float) -> np.ndarray:
    """dot(edge_a, edge_b) / (4 area) (elements.py:60-78)."""
    area = _check_area(area)
    return _one_triangle(2, [p1, p2, p3], area)


def elem_stiff_elastic(p1, p2, p3, area: float, params: ElasticParams) -> np.ndarray:
    """area * B^T C B in the interleaved order (x1, y1, ..., y3) (elements.py:111-154)."""
    area = _check_area(area)
    return _one_triangle(3, [p1, p2, p3], area, lam=params.lam, mu=params.mu)
