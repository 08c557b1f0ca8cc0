"""Seeded jittered/permuted unit-square mesh family used by every benchmark
configuration (BASELINE.json ``configs``).

The reference ships only the fixed-diagonal grid ``generate_unit_square_mesh``
(/root/reference/pkg/src/femasm/mesh.py:147-169) and an unpermuted jitter helper
(/root/reference/pkg/tests/test_assembly.py:35-46).  The BASELINE meshes add a
per-cell coin flip of the diagonal and random vertex / triangle renumbering, so
the generator lives here and feeds the *same* arrays to the oracle and to the
GPU.  It is host-side input preparation, not part of the timed path.

Recipe (draw order is part of the contract, so results are reproducible
bit-for-bit with the same numpy version):

1. grid vertices ``iy*(N+1)+ix`` on ``linspace(0, 1, N+1)``;
2. ``flip = rng.integers(0, 2, N*N)`` per cell; ``flip=0`` splits along
   v00-v11 (the reference diagonal), ``flip=1`` along v10-v01; the two
   triangles of a cell are interleaved, all counterclockwise;
3. interior vertices jittered by ``rng.uniform(-0.2/N, 0.2/N)``;
4. vertex renumbering ``vp = rng.permutation(nq)`` (vertex i becomes vp[i]);
5. triangle renumbering ``tp = rng.permutation(nme)``;
6. vertex weights ``w = rng.uniform(0.5, 2.0, nq)``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["SeededMesh", "seeded_square_mesh", "BASELINE_CONFIGS", "config_by_name"]


@dataclass(frozen=True)
class SeededMesh:
    """Raw arrays of one generated mesh (no validation, no areas)."""

    n: int
    seed: int
    vertices: np.ndarray  # (nq, 2) float64
    connectivity: np.ndarray  # (nme, 3) int64, counterclockwise
    weights: np.ndarray  # (nq,) float64, U(0.5, 2.0)

    @property
    def nq(self) -> int:
        return self.vertices.shape[0]

    @property
    def nme(self) -> int:
        return self.connectivity.shape[0]


def seeded_square_mesh(n: int, seed: int = 0) -> SeededMesh:
    if n < 1:
        raise ValueError(f"n must be >= 1, got {n}")
    rng = np.random.default_rng(seed)
    n1 = n + 1
    nq = n1 * n1
    side = np.linspace(0.0, 1.0, n1)
    verts = np.empty((nq, 2), dtype=np.float64)
    verts[:, 0] = np.tile(side, n1)
    verts[:, 1] = np.repeat(side, n1)

    flip = rng.integers(0, 2, n * n).astype(bool)
    cell = np.arange(n * n, dtype=np.int64)
    iy, ix = np.divmod(cell, n)
    v00 = iy * n1 + ix
    v10 = v00 + 1
    v01 = v00 + n1
    v11 = v01 + 1
    conn = np.empty((2 * n * n, 3), dtype=np.int64)
    first = conn[0::2]
    second = conn[1::2]
    # flip = 0: (v00, v10, v11), (v00, v11, v01);  flip = 1: (v00, v10, v01), (v10, v11, v01)
    first[:, 0] = v00
    first[:, 1] = v10
    first[:, 2] = np.where(flip, v01, v11)
    second[:, 0] = np.where(flip, v10, v00)
    second[:, 1] = v11
    second[:, 2] = v01
    del first, second, flip, cell, iy, ix, v00, v10, v01, v11

    x = verts[:, 0]
    y = verts[:, 1]
    interior = (x > 0) & (x < 1) & (y > 0) & (y < 1)
    verts[interior] += rng.uniform(-0.2 / n, 0.2 / n, size=(int(interior.sum()), 2))

    vp = rng.permutation(nq)
    renumbered = np.empty_like(verts)
    renumbered[vp] = verts
    conn = vp[conn]
    tp = rng.permutation(conn.shape[0])
    conn = conn[tp]
    weights = rng.uniform(0.5, 2.0, nq)
    return SeededMesh(n, seed, renumbered, np.ascontiguousarray(conn), weights)


# BASELINE.json configs: name -> (kind value, N, lam, mu)
BASELINE_CONFIGS = {
    "C1": ("mass", 256, None, None),
    "C2": ("massw", 1024, None, None),
    "C3": ("stiff", 2048, None, None),
    "C4": ("elastic", 2048, 1.0, 0.5),
    "C5": ("stiff", 8192, None, None),
}


def config_by_name(name: str):
    try:
        return BASELINE_CONFIGS[name.upper()]
    except KeyError:
        raise ValueError(f"unknown config {name!r}; expected one of {sorted(BASELINE_CONFIGS)}") from None
