"""CPU oracle for the OptV2 P1 assembly path — TEST INFRASTRUCTURE ONLY.

This module restates, in plain numpy, the algorithm of the reference package ``femasm``
(/root/reference/pkg/src/femasm) for the one path this repository accelerates:
``assemble(mesh, kind, Strategy.OPTV2)``.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s CPU-baseline legs may import it, and only as the checker / the timed CPU
reference.  The product package ``paper_1305_3122_b200`` never imports anything from here.

Pinning: every function is checked against outputs of the real reference produced in the
build container by tests/golden/make_golden.py (small full arrays in tests/golden/*.npz and
SHA-256 digests of the reference output for the BASELINE configurations in
tests/golden/reference_digests.json).  See tests/test_oracle_golden.py.

Arithmetic: numpy evaluates left to right with one rounding per operation; the element
formulas below keep the reference's operation order so values agree bit for bit.  The
triplet->CSC step uses the same numpy primitives as the reference (stable argsort,
sequential ``bincount`` sums) because their exact semantics are the contract.
"""

from __future__ import annotations

import numpy as np

AREA_EPS = 1e-300  # femasm/mesh.py:27

KINDS = ("mass", "massw", "stiff", "elastic")


class OracleDegenerate(ValueError):
    def __init__(self, index, area):
        self.index = int(index)
        self.area = float(area)
        super().__init__(f"triangle {self.index} is degenerate (area={self.area:g})")


def triangle_areas(q: np.ndarray, me: np.ndarray) -> np.ndarray:
    """femasm/mesh.py:51-69 — 0.5*|(x2-x1)(y3-y1) - (x3-x1)(y2-y1)| per triangle."""
    q = np.asarray(q, dtype=np.float64)
    me = np.asarray(me, dtype=np.int64)
    a, b, c = q[me[:, 0]], q[me[:, 1]], q[me[:, 2]]
    cross = (b[:, 0] - a[:, 0]) * (c[:, 1] - a[:, 1]) - (c[:, 0] - a[:, 0]) * (b[:, 1] - a[:, 1])
    return 0.5 * np.abs(cross)


def first_degenerate(areas: np.ndarray):
    """femasm/assembly.py:152-155: index of the first area <= AREA_EPS, or None."""
    bad = np.nonzero(np.asarray(areas) <= AREA_EPS)[0]
    return int(bad[0]) if bad.size else None


def index_pattern(me: np.ndarray, vector: bool):
    """femasm/assembly.py:162-192 — Ig/Jg (r x nme).  Local slot il = a + r_dim*b holds
    element entry (a, b): Ig = dof[a], Jg = dof[b] (column-major element storage)."""
    me = np.asarray(me, dtype=np.int64)
    if vector:
        dofs = np.empty((me.shape[0], 6), dtype=np.int64)
        dofs[:, 0::2] = 2 * me
        dofs[:, 1::2] = 2 * me + 1
    else:
        dofs = me
    rd = dofs.shape[1]
    a_of = np.arange(rd * rd) % rd
    b_of = np.arange(rd * rd) // rd
    return dofs[:, a_of].T.copy(), dofs[:, b_of].T.copy()


def _edges(q, me):
    # femasm/assembly.py:251-254: u = q2 - q3, v = q3 - q1, w = q1 - q2
    p1, p2, p3 = q[me[:, 0]], q[me[:, 1]], q[me[:, 2]]
    return p2 - p3, p3 - p1, p1 - p2


def element_values(kind: str, q, me, areas, w=None, lam=None, mu=None) -> np.ndarray:
    """Kg (r x nme) in the reference's slot order (femasm/assembly.py:214-307)."""
    me = np.asarray(me, dtype=np.int64)
    areas = np.asarray(areas, dtype=np.float64)
    nme = me.shape[0]
    if kind == "mass":  # assembly.py:219-224
        d = areas / 6.0
        o = areas / 12.0
        return np.stack([d if il in (0, 4, 8) else o for il in range(9)])
    if kind == "massw":  # assembly.py:232-242
        tw = np.asarray(w, dtype=np.float64)
        W = [tw[me[:, c]] * areas / 30.0 for c in range(3)]
        low = {
            (0, 0): 3.0 * W[0] + W[1] + W[2],
            (1, 0): W[0] + W[1] + W[2] / 2.0,
            (2, 0): W[0] + W[1] / 2.0 + W[2],
            (1, 1): W[0] + 3.0 * W[1] + W[2],
            (2, 1): W[0] / 2.0 + W[1] + W[2],
            (2, 2): W[0] + W[1] + 3.0 * W[2],
        }
        return np.stack([low[(max(a, b), min(a, b))] for b in range(3) for a in range(3)])
    q = np.asarray(q, dtype=np.float64)
    e = _edges(q, me)
    if kind == "stiff":  # assembly.py:251-263
        four_a = 4.0 * areas
        low = {(a, b): (e[a] * e[b]).sum(axis=1) / four_a for a in range(3) for b in range(a + 1)}
        return np.stack([low[(max(a, b), min(a, b))] for b in range(3) for a in range(3)])
    if kind == "elastic":  # assembly.py:195-211 (gradients) and :278-306
        half_inv = 0.5 / areas
        g = [np.stack([ei[:, 1], -ei[:, 0]]) * half_inv for ei in e]  # g[v] = (gx, gy) rows
        L, M = float(lam), float(mu)
        P = L + 2.0 * M
        out = np.empty((36, nme))
        for j in range(6):
            for i in range(j, 6):
                A, s, B, t = i // 2, i % 2, j // 2, j % 2
                gA, gB = g[A], g[B]
                # the reference's 21 lower rows, written by component pattern (B's gradient first)
                if s == 0 and t == 0:
                    v = (P * gB[0] * gA[0] + M * gB[1] * gA[1]) * areas
                elif s == 1 and t == 1:
                    v = (P * gB[1] * gA[1] + M * gB[0] * gA[0]) * areas
                elif s == 1 and A == B:
                    v = (L * gB[0] * gA[1] + M * gB[0] * gA[1]) * areas
                elif s == 1:
                    v = (L * gB[0] * gA[1] + M * gB[1] * gA[0]) * areas
                else:
                    v = (L * gB[1] * gA[0] + M * gB[0] * gA[1]) * areas
                out[i + 6 * j] = v
                out[j + 6 * i] = v
        return out
    raise ValueError(f"unknown kind {kind!r}")


def matlab_sparse(rows, cols, vals, n_rows: int, n_cols: int):
    """femasm/sparse.py:140-189 — Matlab sparse(I,J,K,m,n) returning CSC arrays
    (col_ptr int64, row_idx int64, values f64): zeros skipped, stable sort of
    col*n_rows+row, left-to-right sums per position (bincount), exact-zero sums dropped."""
    rows = np.asarray(rows, dtype=np.int64).ravel()
    cols = np.asarray(cols, dtype=np.int64).ravel()
    vals = np.asarray(vals, dtype=np.float64).ravel()
    nz = vals != 0.0
    rows, cols, vals = rows[nz], cols[nz], vals[nz]
    key = cols * np.int64(n_rows) + rows
    perm = np.argsort(key, kind="stable")
    key, vals = key[perm], vals[perm]
    if key.size:
        starts = np.ones(key.size, dtype=bool)
        starts[1:] = key[1:] != key[:-1]
        run = np.cumsum(starts) - 1
        sums = np.bincount(run, weights=vals)  # sequential accumulation in sorted order
        pos = key[starts]
        keep = sums != 0.0
        sums, pos = sums[keep], pos[keep]
    else:
        sums = np.zeros(0)
        pos = np.zeros(0, dtype=np.int64)
    out_cols = pos // n_rows
    col_ptr = np.concatenate([[0], np.cumsum(np.bincount(out_cols, minlength=n_cols))]).astype(np.int64)
    return col_ptr, (pos % n_rows).astype(np.int64), sums


def assemble_optv2(kind: str, q, me, areas, w=None, lam=None, mu=None):
    """femasm/assembly.py:400-416 + sparse.py:318-329: OptV2 triplets -> CSC arrays."""
    me = np.asarray(me, dtype=np.int64)
    if kind in ("mass", "stiff", "elastic"):
        bad = first_degenerate(areas)
        if bad is not None:
            raise OracleDegenerate(bad, np.asarray(areas)[bad])
    ig, jg = index_pattern(me, vector=(kind == "elastic"))
    kg = element_values(kind, q, me, areas, w, lam, mu)
    nq = int(np.asarray(q).shape[0]) if q is not None else int(me.max()) + 1
    n = 2 * nq if kind == "elastic" else nq
    # column-major flatten: slot k*r + il is triangle k, local il (sparse.py:318-325)
    return matlab_sparse(ig.ravel(order="F"), jg.ravel(order="F"), kg.ravel(order="F"), n, n)


def assemble_row_block(kind: str, q, me, areas, w, lam, mu, v0: int, v1: int):
    """Row-block subset oracle: assemble only the triangles touching
    vertex rows [v0, v1) (triangle order preserved, so per-position sums are unchanged)
    and return the CSR/CSC slice of those rows as (ptr local, idx, vals)."""
    me = np.asarray(me, dtype=np.int64)
    touch = ((me >= v0) & (me < v1)).any(axis=1)
    sub_me = me[touch]
    sub_areas = np.asarray(areas)[touch]
    ptr, idx, vals = assemble_optv2(kind, q, sub_me, sub_areas, w, lam, mu)
    rpv = 2 if kind == "elastic" else 1
    c0, c1 = rpv * v0, rpv * v1
    lo, hi = ptr[c0], ptr[c1]
    return ptr[c0:c1 + 1] - lo, idx[lo:hi], vals[lo:hi]


def assemble_seeded(kind: str, mesh, lam=1.0, mu=0.5):
    """Convenience: assemble a meshgen.SeededMesh with its own areas / weights."""
    areas = triangle_areas(mesh.vertices, mesh.connectivity)
    return assemble_optv2(kind, mesh.vertices, mesh.connectivity, areas, mesh.weights, lam, mu)
