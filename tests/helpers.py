"""Shared test helpers (digests, seeded meshes, CSR comparison)."""

from __future__ import annotations

import hashlib

import numpy as np


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def csc_digests(col_ptr, row_idx, values):
    return (
        digest(np.asarray(col_ptr).astype("<i8")),
        digest(np.asarray(row_idx).astype("<i8")),
        digest(np.asarray(values).astype("<f8")),
    )


def mesh_digest(sm) -> str:
    return digest(sm.vertices.astype("<f8"), sm.connectivity.astype("<i8"), sm.weights.astype("<f8"))


def assert_same_csc(got, ref, what=""):
    gp, gi, gv = (np.asarray(x) for x in got)
    rp, ri, rv = (np.asarray(x) for x in ref)
    assert np.array_equal(gp.astype(np.int64), rp.astype(np.int64)), f"{what}: pointer arrays differ"
    assert np.array_equal(gi.astype(np.int64), ri.astype(np.int64)), f"{what}: index arrays differ"
    assert gv.shape == rv.shape, f"{what}: value counts differ"
    # bitwise (the contract allows 1e-12 relative; the design delivers 0)
    assert np.array_equal(gv.view(np.int64), rv.view(np.int64)), (
        f"{what}: values differ, max rel {np.abs(gv - rv).max() / max(np.abs(rv).max(), 1e-300):.3e}")


def rel_err(got_vals, ref_vals) -> float:
    ref = np.asarray(ref_vals)
    scale = np.abs(ref).max() if ref.size else 1.0
    return float(np.abs(np.asarray(got_vals) - ref).max() / scale) if ref.size else 0.0


def csr_digests_device(rowptr, col, val, chunk=1 << 26):
    """SHA-256 of device CSR arrays in femasm's CSC dtypes (int64, int64, f64), streamed to the
    host in chunks (the C5 matrix does not need a second full host copy)."""
    import torch

    out = []
    for t, dt in ((rowptr, torch.int64), (col, torch.int64), (val, torch.float64)):
        h = hashlib.sha256()
        for s in range(0, t.numel(), chunk):
            h.update(np.ascontiguousarray(t[s:s + chunk].to(dt).cpu().numpy()).astype(
                "<i8" if dt is torch.int64 else "<f8", copy=False).tobytes())
        out.append(h.hexdigest())
    return tuple(out)
