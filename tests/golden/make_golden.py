"""Generate the golden fixtures by running the REAL reference package (femasm) in the build
container, where /root/reference exists.  The GPU box never runs this script: it only reads
the committed outputs.

    python tests/golden/make_golden.py small           -> tests/golden/small_cases.npz
    python tests/golden/make_golden.py digests C1 C2   -> tests/golden/reference_digests.json
    python tests/golden/make_golden.py digests C5ALL    -> every C5 row block + the whole C5 digest
    python tests/golden/make_golden.py loops           -> tests/golden/loop_cases.npz
    python tests/golden/make_golden.py mesh_text       -> tests/golden/mesh_text_cases.json

small_cases.npz: seeded BASELINE-family meshes (tiny N), the reference's own generators
(square / disk) and the reference's OptV2 output for every kind, as full arrays.
reference_digests.json: SHA-256 of the reference's CSC arrays for the BASELINE configs
(seeds 0..2), so full-size parity on the GPU box is checked against the reference itself.
"""

from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parents[1]
sys.path.insert(0, str(REPO))
sys.path.insert(0, "/root/reference/pkg/src")

import femasm  # noqa: E402  (the reference, read-only)

from paper_1305_3122_b200.meshgen import BASELINE_CONFIGS, seeded_square_mesh  # noqa: E402

KIND = {
    "mass": femasm.MatrixKind.MASS,
    "massw": femasm.MatrixKind.WEIGHTED_MASS,
    "stiff": femasm.MatrixKind.STIFFNESS,
    "elastic": femasm.MatrixKind.ELASTIC,
}


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def mesh_digest(m) -> str:
    return digest(m.vertices.astype("<f8"), m.connectivity.astype("<i8"), m.weights.astype("<f8"))


def ref_assemble(V, C, kind, w=None, lam=1.0, mu=0.5):
    mesh = femasm.Mesh(V, C)
    kw = {}
    if kind == "massw":
        tw = np.asarray(w, dtype=np.float64)
        kw["weight"] = femasm.WeightField("samples", lambda x, y: tw)
    if kind == "elastic":
        kw["params"] = femasm.ElasticParams(lam, mu)
    m = femasm.assemble(mesh, KIND[kind], femasm.Strategy.OPTV2, **kw)
    return mesh, m


def small():
    out = {}
    cases = []
    for n in (2, 5, 16):
        for seed in (0, 1):
            sm = seeded_square_mesh(n, seed)
            name = f"seeded_n{n}_s{seed}"
            out[f"{name}/V"] = sm.vertices
            out[f"{name}/C"] = sm.connectivity
            out[f"{name}/w"] = sm.weights
            for kind in KIND:
                lam, mu = (2.0, 0.7) if seed == 1 else (1.0, 0.5)
                mesh, m = ref_assemble(sm.vertices, sm.connectivity, kind, sm.weights, lam, mu)
                out[f"{name}/{kind}/col_ptr"] = m.col_ptr
                out[f"{name}/{kind}/row_idx"] = m.row_idx
                out[f"{name}/{kind}/values"] = m.values
                out[f"{name}/{kind}/lam_mu"] = np.array([lam, mu])
            out[f"{name}/areas"] = mesh.areas
            # batch kernels of the reference on the same mesh
            out[f"{name}/kg_stiff"] = femasm.batch_kg_stiff(mesh)
            out[f"{name}/kg_elastic"] = femasm.batch_kg_elastic(mesh, femasm.ElasticParams(1.0, 0.5))
            out[f"{name}/kg_massw"] = femasm.batch_kg_mass_weighted(
                mesh, femasm.WeightField("samples", lambda x, y, w=sm.weights: w))
            out[f"{name}/kg_mass"] = femasm.batch_kg_mass(mesh.areas)
            g = femasm.batch_gradients(mesh)
            out[f"{name}/grad"] = np.concatenate([g.g1, g.g2, g.g3])
            cases.append(name)
    # the reference's own structured generators, with its test defaults
    gens = {
        "square_n4": femasm.generate_unit_square_mesh(4),
        "square_n1": femasm.generate_unit_square_mesh(1),
        "disk_n4": femasm.generate_disk_mesh(4),
        "disk_n6": femasm.generate_disk_mesh(6),
    }
    for name, mesh in gens.items():
        out[f"{name}/V"] = mesh.vertices
        out[f"{name}/C"] = mesh.connectivity
        out[f"{name}/areas"] = mesh.areas
        for kind in KIND:
            kw = {}
            if kind == "massw":
                kw["weight"] = femasm.WeightField.quadratic()
            if kind == "elastic":
                kw["params"] = femasm.ElasticParams(1.0, 1.0)
            m = femasm.assemble(mesh, KIND[kind], femasm.Strategy.OPTV2, **kw)
            out[f"{name}/{kind}/col_ptr"] = m.col_ptr
            out[f"{name}/{kind}/row_idx"] = m.row_idx
            out[f"{name}/{kind}/values"] = m.values
    np.savez_compressed(HERE / "small_cases.npz", **out)
    print("small cases:", cases + list(gens))


def loops():
    """Element-loop strategies (CLASSICAL, OPTV0, OPTV1; assembly.py:359-397) and the
    per-element API elem_* (elements.py:34-154) of the reference, as full arrays ->
    tests/golden/loop_cases.npz.  The reference builds CLASSICAL/OPTV0 with CscBuilder
    (explicit zeros kept) and every strategy with the per-element formulas, so the bits differ
    from OPTV2's; the meshes are small because the reference's CscBuilder is O(nnz) per
    insertion."""
    out = {}
    rng = np.random.default_rng(7)
    # elem_*: random triangles (counterclockwise, well shaped), weights, Lame parameters
    P = rng.uniform(-1.0, 1.0, (64, 3, 2))
    P[:, 1] = P[:, 0] + rng.uniform(0.2, 1.0, (64, 2)) * [1.0, 0.1]
    P[:, 2] = P[:, 0] + rng.uniform(0.2, 1.0, (64, 2)) * [0.1, 1.0]
    A = femasm.compute_areas(P.reshape(-1, 2), np.arange(192).reshape(64, 3))
    W = rng.uniform(0.5, 2.0, (64, 3))
    out["elem/P"], out["elem/A"], out["elem/W"] = P, A, W
    params = femasm.ElasticParams(1.3, 0.4)
    out["elem/lam_mu"] = np.array([1.3, 0.4])
    out["elem/mass"] = np.stack([femasm.elem_mass(a) for a in A])
    out["elem/massw"] = np.stack([femasm.elem_mass_weighted(a, *w) for a, w in zip(A, W)])
    out["elem/stiff"] = np.stack([femasm.elem_stiff(p[0], p[1], p[2], a) for p, a in zip(P, A)])
    out["elem/elastic"] = np.stack([femasm.elem_stiff_elastic(p[0], p[1], p[2], a, params) for p, a in zip(P, A)])
    meshes = {
        "square_n4": femasm.generate_unit_square_mesh(4),
        "disk_n4": femasm.generate_disk_mesh(4),
        "seeded_n5_s1": femasm.Mesh(seeded_square_mesh(5, 1).vertices, seeded_square_mesh(5, 1).connectivity),
    }
    for name, mesh in meshes.items():
        out[f"{name}/V"] = mesh.vertices
        out[f"{name}/C"] = mesh.connectivity
        for kind in KIND:
            kw = {}
            if kind == "massw":
                kw["weight"] = femasm.WeightField.quadratic()
            if kind == "elastic":
                kw["params"] = femasm.ElasticParams(2.0, 0.7)
            for strat in ("CLASSICAL", "OPTV0", "OPTV1"):
                m = femasm.assemble(mesh, KIND[kind], getattr(femasm.Strategy, strat), **kw)
                for f in ("col_ptr", "row_idx", "values"):
                    out[f"{name}/{kind}/{strat}/{f}"] = getattr(m, f)
    np.savez_compressed(HERE / "loop_cases.npz", **out)
    print("loop cases:", list(meshes))


MESH_TEXT_CASES = {
    "plain": "3 1\n0 0\n1 0\n0 1\n1 2 3\n",
    "crlf_tabs_blank_tail": "3 1\r\n0\t0\r\n1.5e0 -0\r\n.25   1.\r\n1 2 3\r\n\r\n   \r\n",
    "python_tokens": "3 1\n+0 0\n1_0 0\ninf 1\n+1 0_2 3\n",
    "empty": "",
    "blank_header": "  \n3 1\n",
    "header_fields": "3\n0 0\n",
    "header_int": "3 x\n",
    "counts": "0 1\n",
    "short": "3 1\n0 0\n1 0\n",
    "coords_count": "3 1\n0 0\n1 0 0\n0 1\n1 2 3\n",
    "coord_value": "3 1\n0 0\n1 zz\n0 1\n1 2 3\n",
    "tri_fields": "3 1\n0 0\n1 0\n0 1\n1 2\n",
    "tri_int": "3 1\n0 0\n1 0\n0 1\n1 2 3.0\n",
    "tri_range": "3 1\n0 0\n1 0\n0 1\n1 2 4\n",
    "trailing": "3 1\n0 0\n1 0\n0 1\n1 2 3\n\nextra\n",
    "invalid_mesh": "3 1\n0 0\n1 0\n0 1\n1 1 3\n",
    "degenerate": "3 1\n0 0\n1 0\n2 0\n1 2 3\n",
    "hex_float": "3 1\n0x1p0 0\n1 0\n0 1\n1 2 3\n",
    "form_feed": "3 1\n0 0\n1 0\f\n0 1\n1 2 3\n",
}


def mesh_text():
    """femasm.read_mesh on small text files -> tests/golden/mesh_text_cases.json: the arrays it
    returns or the MeshFormatError (line number and message, path replaced by '<path>')."""
    import tempfile

    out = {}
    d = Path(tempfile.mkdtemp())
    for name, text in MESH_TEXT_CASES.items():
        p = d / f"{name}.txt"
        p.write_bytes(text.encode("ascii"))
        try:
            m = femasm.read_mesh(p)
            out[name] = {"text": text, "ok": True, "vertices": m.vertices.tolist(),
                         "connectivity": m.connectivity.tolist()}
        except femasm.MeshFormatError as exc:
            out[name] = {"text": text, "ok": False, "line_no": exc.line_no,
                         "message": str(exc).replace(str(p), "<path>")}
    (HERE / "mesh_text_cases.json").write_text(json.dumps(out, indent=1, sort_keys=True))
    print("mesh text cases:", {k: v["ok"] for k, v in out.items()})


def digests(names):
    path = HERE / "reference_digests.json"
    data = json.loads(path.read_text()) if path.exists() else {}
    for spec in names:
        # spec: C1 | C1:s1 | EL64 (elastic lam=2 mu=0.7 N=64 seed 0) | C5B:G:b (row block b of G)
        if spec == "C5ALL":
            c5_all_blocks(data, path)
            continue
        if spec.startswith("C5B"):
            _, g, blk = spec.split(":")
            row_block_digest(data, path, "C5", int(g), int(blk), seed=0)
            continue
        if spec.startswith("EL64"):
            kind, n, lam, mu, seeds = "elastic", 64, 2.0, 0.7, [0]
            cfg = "EL64"
        else:
            cfg, _, s = spec.partition(":")
            kind, n, lam, mu = BASELINE_CONFIGS[cfg]
            seeds = [int(s[1:])] if s else [0, 1, 2]
            lam = 1.0 if lam is None else lam
            mu = 0.5 if mu is None else mu
        for seed in seeds:
            t0 = time.perf_counter()
            sm = seeded_square_mesh(n, seed)
            mesh, m = ref_assemble(sm.vertices, sm.connectivity, kind, sm.weights, lam, mu)
            t1 = time.perf_counter()
            key = f"{cfg}/s{seed}"
            data[key] = {
                "kind": kind, "N": n, "seed": seed, "lam": lam, "mu": mu,
                "nq": int(sm.nq), "nme": int(sm.nme), "nnz": int(m.nnz),
                "mesh_sha256": mesh_digest(sm),
                "areas_sha256": digest(mesh.areas.astype("<f8")),
                "col_ptr_sha256": digest(m.col_ptr.astype("<i8")),
                "row_idx_sha256": digest(m.row_idx.astype("<i8")),
                "values_sha256": digest(m.values.astype("<f8")),
                "values_sum": float(m.values.sum()),
                "reference_seconds": round(t1 - t0, 2),
            }
            print(key, data[key]["nnz"], f"{t1 - t0:.1f}s", flush=True)
            path.write_text(json.dumps(data, indent=1, sort_keys=True))
            del mesh, m, sm


def c5_all_blocks(data, path, cfg="C5", seed=0, G=16):
    """Every row block of the G-way split of `cfg`, from ONE generated mesh, each assembled by
    femasm through the row-block subset (as row_block_digest).  The block arrays are also fed,
    in row order, into streaming SHA-256s of every coarser split G/2, G/4, ..., 1 (block b of
    G/2 is blocks 2b, 2b+1 of G, because floor(nq*b/(G/2)) == floor(nq*2b/G)), so the digests
    of the whole matrix (G=1, what a single GPU assembles) and of the G=8 split come out of
    femasm runs that each fit in memory."""
    kind, n, lam, mu = BASELINE_CONFIGS[cfg]
    t0 = time.perf_counter()
    sm = seeded_square_mesh(n, seed)
    nq = sm.nq
    C = sm.connectivity
    levels = []
    g = G
    while g >= 1:
        levels.append(g)
        g //= 2
    hs = {g: None for g in levels}
    state = {g: {"blk": -1, "h": None, "lo": 0, "nnz": 0, "touched": 0} for g in levels}
    mdig = mesh_digest(sm)

    def close(g):
        st = state[g]
        if st["h"] is None:
            return
        b = st["blk"]
        v0, v1 = (nq * b) // g, (nq * (b + 1)) // g
        key = f"{cfg}B/s{seed}/G{g}/b{b}" if g > 1 else f"{cfg}/s{seed}"
        hp, hr, hv, vs = st["h"]
        ent = {"kind": kind, "N": n, "seed": seed, "nq": int(nq), "nme": int(sm.nme),
               "nnz": int(st["nnz"]), "mesh_sha256": mdig,
               "col_ptr_sha256": hp.hexdigest(), "row_idx_sha256": hr.hexdigest(),
               "values_sha256": hv.hexdigest(), "via": f"streamed from the G={G} row-block subsets"}
        if g > 1:
            ent.update({"G": g, "block": b, "v0": int(v0), "v1": int(v1)})
        else:
            ent.update({"lam": lam, "mu": mu, "values_sum_blocks": vs})
        data[key] = ent
        print(key, ent["nnz"], flush=True)

    for blk in range(G):
        v0, v1 = (nq * blk) // G, (nq * (blk + 1)) // G
        touch = ((C >= v0) & (C < v1)).any(axis=1)
        sub = femasm.Mesh(sm.vertices, C[touch])
        m = femasm.assemble(sub, KIND[kind], femasm.Strategy.OPTV2)
        lo, hi = int(m.col_ptr[v0]), int(m.col_ptr[v1])
        ptr = (m.col_ptr[v0:v1 + 1] - lo).astype("<i8")
        rows = m.row_idx[lo:hi].astype("<i8")
        vals = m.values[lo:hi].astype("<f8")
        del m, sub
        for g in levels:
            b = blk * g // G
            st = state[g]
            if st["blk"] != b:
                close(g)
                st.update(blk=b, h=(hashlib.sha256(), hashlib.sha256(), hashlib.sha256(), 0.0), lo=0, nnz=0)
                st["h"][0].update(np.zeros(1, "<i8").tobytes())
            hp, hr, hv, vs = st["h"]
            hp.update((ptr[1:] + st["nnz"]).tobytes())
            hr.update(rows.tobytes())
            hv.update(vals.tobytes())
            st["h"] = (hp, hr, hv, vs + float(vals.sum()))
            st["nnz"] += len(rows)
        print(f"block {blk}/{G} rows [{v0},{v1}) nnz {len(rows)} {time.perf_counter() - t0:.0f}s", flush=True)
        del ptr, rows, vals
    for g in levels:
        close(g)
    path.write_text(json.dumps(data, indent=1, sort_keys=True))


def row_block_digest(data, path, cfg, G, blk, seed=0):
    """Reference output restricted to vertex rows [v0, v1) of block blk of G, obtained with
    the row-block subset: the triangles touching the block, in their
    original order, assembled by femasm; the block's CSC columns equal the full assembly's."""
    kind, n, lam, mu = BASELINE_CONFIGS[cfg]
    t0 = time.perf_counter()
    sm = seeded_square_mesh(n, seed)
    nq = sm.nq
    v0, v1 = (nq * blk) // G, (nq * (blk + 1)) // G
    C = sm.connectivity
    touch = ((C >= v0) & (C < v1)).any(axis=1)
    sub = femasm.Mesh(sm.vertices, C[touch])
    m = femasm.assemble(sub, KIND[kind], femasm.Strategy.OPTV2)
    lo, hi = int(m.col_ptr[v0]), int(m.col_ptr[v1])
    ptr = m.col_ptr[v0:v1 + 1] - lo
    key = f"{cfg}B/s{seed}/G{G}/b{blk}"
    data[key] = {
        "kind": kind, "N": n, "seed": seed, "G": G, "block": blk, "v0": int(v0), "v1": int(v1),
        "nq": int(nq), "nme": int(sm.nme), "touched": int(touch.sum()), "nnz": int(hi - lo),
        "mesh_sha256": mesh_digest(sm),
        "col_ptr_sha256": digest(ptr.astype("<i8")),
        "row_idx_sha256": digest(m.row_idx[lo:hi].astype("<i8")),
        "values_sha256": digest(m.values[lo:hi].astype("<f8")),
        "reference_seconds": round(time.perf_counter() - t0, 2),
    }
    print(key, data[key]["nnz"], data[key]["reference_seconds"], flush=True)
    path.write_text(json.dumps(data, indent=1, sort_keys=True))


if __name__ == "__main__":
    if sys.argv[1] == "small":
        small()
    elif sys.argv[1] == "loops":
        loops()
    elif sys.argv[1] == "mesh_text":
        mesh_text()
    elif sys.argv[1] == "digests":
        digests(sys.argv[2:])
