#!/usr/bin/env python
"""Benchmark of the B200 OptV2 P1 assembly (one JSON line on rank 0).

Metric (BASELINE.json): triangles assembled per second, device-timed, including the CSR
build, plus achieved HBM GB/s.  Workload (default): BASELINE configs[4] = C5, the P1 stiffness
matrix on the seeded jittered/permuted unit-square mesh with N=8192 (134,217,728 triangles,
67,125,249 vertices, ~470 M stored entries) - the largest configuration that fits one GPU.
C1-C4 via --config (they are parity-test cases, not headline lines).

One step = one complete OptV2 assembly from device-resident inputs: plan build (part
histogram, part placement, per-part vertex sort) + fused row kernel writing rowptr/col/val,
i.e. the reference's `assemble(mesh, kind, OPTV2)` with nothing cached between steps
("cold").  The L2 is flushed (a 512 MB buffer is zeroed) between timed steps, outside the
timed windows.  After the timed loop the last step's CSR is hashed and compared with the
SHA-256 digests of femasm's own output for the same seeded mesh (tests/golden/
reference_digests.json, produced by running the reference): the line carries the verdict.
N > 1 (torchrun): rank g assembles the matrix rows of vertex block g (row-block
decomposition); the step includes the NCCL allgather of the per-rank nnz
that yields the global row offsets.  The total work is fixed: "scaling": "strong".

CPU legs (test infrastructure never on the measured GPU path):
  * cpu_baseline (rank 0, N=1): femasm itself (the unmodified reference, installed offline
    into baseline/_ref; the numpy restatement in oracle/ if that install is missing) on ONE
    core, timed like femasm bench._time_cell (/root/reference/pkg/src/femasm/bench.py:97-122:
    one discarded warm-up, median of the timed runs) on a bounded sample: the sub-mesh made of
    the triangles touching one block of vertex rows (vertices compacted), a few million
    triangles; femasm OptV2 is linear in nme, so its triangles/s is reported
    as the full-mesh rate, labelled extrapolated.
  * --impl reference: the same femasm call on every host core (one row-block sub-mesh per
    process per step), rank 0 only.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

import numpy as np  # noqa: E402

METRIC = "triangles assembled/sec (device-timed, incl. CSR build)"
UNIT = "triangles/s"
DEFAULT_CONFIG = "C5"
DESCR = {
    "C1": "P1 mass, N=256 seeded jittered/permuted unit square",
    "C2": "P1 weighted mass (vertex weights U(0.5,2)), N=1024 seeded jittered/permuted unit square",
    "C3": "P1 stiffness, N=2048 seeded jittered/permuted unit square",
    "C4": "2D linear elasticity lam=1 mu=0.5, N=2048 seeded jittered/permuted unit square",
    "C5": "P1 stiffness, N=8192 seeded jittered/permuted unit square (largest config on one GPU)",
}
DIGESTS = REPO / "tests" / "golden" / "reference_digests.json"
REF_INSTALL = REPO / "baseline" / "_ref"


def launches_per_step(kind, nme, nq, nv):
    """Our kernels launched per cold step (fa_assemble_cold); memsets are not counted.  The
    two-level plan rule mirrors fa_plan_create (more than 8192 parts of 1024 rows, or more than
    160 MB of part records with more than 256 parts) and adds k_part_split."""
    nparts = -(-nv // 1024)
    two_level = nparts > 8192 or (48 * nme // max(nq, 1) * nv > (160 << 20) and nparts > 256)
    hist = "k_part_hist (weighted mass: also the per-triangle W records)" if kind == "massw" else "k_part_hist"
    return (["k_reset", hist, "k_part_scan", "k_part_place"] + (["k_part_split"] if two_level else [])
            + ["k_part_sort", "k_reset", "k_rows", "k_compact (exits at once unless a sum was exactly zero)"])


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default=DEFAULT_CONFIG)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--cpu-baseline-runs", type=int, default=2, help="timed runs of the 1-core CPU baseline (0: skip)")
    ap.add_argument("--e2e-steps", type=int, default=16)
    ap.add_argument("--graph", type=int, default=1, help="replay each step as a captured CUDA graph (N=1)")
    ap.add_argument("--verify", type=int, default=1, help="hash the last step's CSR against femasm's digests")
    ap.add_argument("--ref-budget-s", type=float, default=150.0,
                    help="--impl reference: wall-clock budget of the timed steps (sizes each step's sample)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def mesh_for(config: str, seed: int):
    from paper_1305_3122_b200.meshgen import BASELINE_CONFIGS, seeded_square_mesh

    kind, n, lam, mu = BASELINE_CONFIGS[config]
    sm = seeded_square_mesh(n, seed)
    return kind, n, (1.0 if lam is None else lam), (0.5 if mu is None else mu), sm


def common_config(config, seed, sm):
    """`config` of both arms (identical, so the driver compares like with like)."""
    return {"workload": f"{config}: {DESCR[config]}", "nq": sm.nq, "nme": sm.nme, "seed": seed,
            "l2": "inputs (me 12 B/tri + q 16 B/vertex) and the CSR exceed L2 at C3-C5; a 512 MB buffer is "
                  "also zeroed between timed GPU steps (outside the timed windows)"}


def alg_bytes(kind, nme, nq, n_rows, nnz):
    """Compulsory bytes of the paper-level API: me int32 + areas read once,
    q (stiffness, elasticity) or w (weighted mass) read once, rowptr + col int32 + val f64
    written once."""
    b = 12 * nme + 8 * nme
    if kind in ("stiff", "elastic"):
        b += 16 * nq
    if kind == "massw":
        b += 8 * nq
    return b + 8 * (n_rows + 1) + 12 * nnz


class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region (B200_PROFILING.md).

    A background thread issues single-shot queries back to back; every sample is timestamped
    and the summary keeps the samples taken inside [mark_start, mark_end].  When the timed
    region is shorter than one query, the samples adjacent to it are reported and flagged."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, gpu_index: int):
        import threading

        self.gpu = gpu_index
        self.samples = []  # (t_mid, sm, smax, reasons)
        self.stop_evt = threading.Event()
        self.thread = threading.Thread(target=self._run, daemon=True)
        self.t0 = self.t1 = None
        self.ok = True

    def _query(self):
        t_a = time.perf_counter()
        try:
            out = subprocess.run(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                                  "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5).stdout
        except (OSError, subprocess.SubprocessError):
            self.ok = False
            return
        t_b = time.perf_counter()
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm, smax = float(parts[1]), float(parts[2])
            except ValueError:
                continue
            reasons = {nm for nm, val in zip(self.NAMES, parts[5:9]) if val.lower() == "active"}
            self.samples.append(((t_a + t_b) / 2, sm, smax, reasons))

    def _run(self):
        while not self.stop_evt.is_set() and self.ok:
            self._query()

    def start(self):
        self.thread.start()
        deadline = time.perf_counter() + 10
        while not self.samples and self.ok and time.perf_counter() < deadline:
            time.sleep(0.01)

    def mark_start(self):
        self.t0 = time.perf_counter()

    def mark_end(self):
        self.t1 = time.perf_counter()

    def stop(self):
        self.stop_evt.set()
        self.thread.join(timeout=10)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        inside = [s for s in self.samples if self.t0 <= s[0] <= self.t1]
        note = "sampled inside the timed region"
        if not inside:  # region shorter than a query: the samples just before and after it
            before = [s for s in self.samples if s[0] < self.t0][-1:]
            after = [s for s in self.samples if s[0] > self.t1][:1]
            inside = before + after
            note = "timed region shorter than one nvidia-smi query: adjacent samples"
        reasons = set().union(*(s[3] for s in inside)) if inside else set()
        return {"sm_mhz": statistics.median(s[1] for s in inside), "sm_max_mhz": max(s[2] for s in inside),
                "reasons": sorted(reasons), "samples": len(inside), "note": note}


def measured_peak():
    p = REPO / "MEASURED_PEAKS.json"
    try:
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def ncu_traffic(config: str):
    """DRAM bytes per row-kernel launch from the committed ncu --set full capture, if any."""
    p = REPO / "profiles" / "ncu_summary.json"
    try:
        d = json.loads(p.read_text())
        e = d["configs"][config]["k_rows"]
        return float(e["dram_bytes_read"]) + float(e["dram_bytes_write"])
    except Exception:
        return None


# ------------------------------------------------------------------------------------------
# CPU legs: femasm (the reference) on a bounded row-block sample
# ------------------------------------------------------------------------------------------
def reference_module():
    """femasm from the offline install in baseline/_ref (the unmodified reference package), or
    None when it is absent (then the numpy restatement in oracle/ stands in)."""
    if REF_INSTALL.is_dir() and str(REF_INSTALL) not in sys.path:
        sys.path.insert(0, str(REF_INSTALL))
    try:
        import femasm  # noqa: F401

        return femasm
    except ImportError:
        return None


def row_block_sample(sm, G, b):
    """The sub-mesh of the triangles touching vertex rows [v0, v1) (block b of G), in their
    original order, with the used vertices compacted (order-preserving renumbering, so the
    sort structure of OptV2 is unchanged).  Returns (V, C, w, v0, v1)."""
    v0, v1 = (sm.nq * b) // G, (sm.nq * (b + 1)) // G
    C = sm.connectivity
    touch = ((C >= v0) & (C < v1)).any(axis=1)
    sub = C[touch]
    used = np.unique(sub)
    return sm.vertices[used], np.searchsorted(used, sub), sm.weights[used], v0, v1


def sample_split(kind, nme, target_tri):
    """Smallest power-of-two row split whose block sub-mesh has at most ~target_tri triangles
    (a block of 1/G of the rows touches about 1 - (1 - 1/G)^3 of the triangles)."""
    G = 1
    while nme * (1 - (1 - 1 / G) ** 3) > target_tri and G < (1 << 20):
        G *= 2
    return G


def _femasm_args(femasm, kind, w, lam, mu):
    KIND = {"mass": femasm.MatrixKind.MASS, "massw": femasm.MatrixKind.WEIGHTED_MASS,
            "stiff": femasm.MatrixKind.STIFFNESS, "elastic": femasm.MatrixKind.ELASTIC}
    kw = {}
    if kind == "massw":
        tw = np.asarray(w, dtype=np.float64)
        kw["weight"] = femasm.WeightField("samples", lambda x, y: tw)
    if kind == "elastic":
        kw["params"] = femasm.ElasticParams(lam, mu)
    return KIND[kind], kw


def cpu_assembler(kind, V, C, w, lam, mu):
    """A zero-argument callable running one OptV2 assembly of (V, C) on the host (femasm, or
    the restatement), plus the kind label.  Mesh construction is outside the callable, as in
    femasm bench (/root/reference/pkg/src/femasm/bench.py:157-159)."""
    femasm = reference_module()
    if femasm is not None:
        mesh = femasm.Mesh(V, C)
        mk, kw = _femasm_args(femasm, kind, w, lam, mu)
        return (lambda: femasm.assemble(mesh, mk, femasm.Strategy.OPTV2, **kw)), "reference", "femasm (baseline/_ref)"
    from oracle import femasm_oracle as fo

    areas = fo.triangle_areas(V, C)
    return (lambda: fo.assemble_optv2(kind, V, C, areas, w, lam, mu)), "port", "numpy restatement of femasm (oracle/)"


def cpu_baseline(config, kind, sm, lam, mu, runs):
    """1-core reference baseline on a bounded sample (about 10-30 s of CPU work)."""
    target = 8e5 if kind == "elastic" else 3e6
    G = sample_split(kind, sm.nme, target)
    V, C, w, v0, v1 = row_block_sample(sm, G, 0)
    fn, kind_label, what = cpu_assembler(kind, V, C, w, lam, mu)
    times = []
    for i in range(runs + 1):  # run 0 is the discarded warm-up (femasm bench._time_cell)
        t0 = time.perf_counter()
        fn()
        dt = time.perf_counter() - t0
        if i > 0:
            times.append(dt)
    t = statistics.median(times)
    sample = (f"{what} OptV2, 1 thread, on the sub-mesh of the {config} mesh made of the {len(C)} triangles touching "
              f"vertex rows [{v0}, {v1}) (block 0 of {G}; {len(V)} vertices compacted), median of {runs} after 1 "
              f"discarded warm-up (femasm bench._time_cell); triangles/s extrapolated linearly to the full "
              f"{sm.nme}-triangle mesh (OptV2 is linear in nme, SURVEY.md §8(d))"
              if G > 1 else
              f"{what} OptV2, 1 thread, full {config} mesh ({sm.nme} triangles), median of {runs} after 1 warm-up")
    return {"value": len(C) / t, "unit": UNIT, "cores": 1, "kind": kind_label, "sample": sample,
            "seconds_per_sample": t, "sample_triangles": int(len(C)), "extrapolated": G > 1}


_REF = {}


def _ref_block(b):
    d = _REF
    V, C, w, _, _ = row_block_sample(d["sm"], d["G"], b)
    fn, _, _ = cpu_assembler(d["kind"], V, C, w, d["lam"], d["mu"])
    t0 = time.perf_counter()
    fn()
    return len(C), time.perf_counter() - t0


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    import multiprocessing as mp

    kind, n, lam, mu, sm = mesh_for(args.config, args.seed)
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    femasm = reference_module()
    # per-process sample sized so the K + W steps fit the budget (femasm: ~3e5 scalar /
    # ~8e4 elastic triangles per second per core)
    rate = 3e4 if kind == "elastic" else 1.2e5  # per process with every core busy (measured on the box)
    per_step_s = max(0.5, args.ref_budget_s / max(1, args.steps + args.warmup))
    G = max(sample_split(kind, sm.nme, rate * per_step_s), 1)
    while G < cores:
        G *= 2
    procs = min(cores, G)
    _REF.update(kind=kind, sm=sm, G=G, lam=lam, mu=mu)
    ctx = mp.get_context("fork")
    times, tris = [], []
    with ctx.Pool(procs) as pool:
        for i in range(args.warmup + args.steps):
            blocks = [(i * procs + j) % G for j in range(procs)]
            t0 = time.perf_counter()
            out = pool.map(_ref_block, blocks)
            dt = time.perf_counter() - t0
            if i >= args.warmup:
                times.append(dt)
                tris.append(sum(c for c, _ in out))
    total = sum(times)
    value = sum(tris) / total
    label = "reference" if femasm is not None else "port"
    what = "femasm (baseline/_ref)" if femasm is not None else "numpy restatement of femasm (oracle/)"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total / len(times) * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic: seeded jittered/permuted unit-square mesh (SURVEY.md §8(d)), seed {args.seed}",
        "config": common_config(args.config, args.seed, sm),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": procs, "kind": label,
                         "sample": f"{what} OptV2 in {procs} host processes; each step = {procs} distinct row-block "
                                   f"sub-meshes of the {G}-way split (triangles touching the block's vertex rows, "
                                   f"vertices compacted), ~{int(np.mean(tris)) if tris else 0} triangles per step; "
                                   "value = triangles assembled / step wall time"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------------------
# parity of the timed output: SHA-256 against femasm's own digests
# ------------------------------------------------------------------------------------------
def csr_digests(rowptr, col, val, chunk=1 << 26):
    """SHA-256 of (rowptr int64, col as int64, val f64) in femasm's CSC dtypes (the matrices
    are bitwise symmetric, so CSR == CSC), streamed from the device in chunks."""
    import torch

    out = []
    for t, conv in ((rowptr, torch.int64), (col, torch.int64), (val, torch.float64)):
        h = hashlib.sha256()
        for s in range(0, t.numel(), chunk):
            h.update(t[s:s + chunk].to(conv).cpu().numpy().astype(
                "<i8" if conv is torch.int64 else "<f8", copy=False).tobytes())
        out.append(h.hexdigest())
    return out


def verify_output(config, seed, world, rank, rowptr, col, val, nnz, mesh_sha):
    """Compare the last timed step's CSR with femasm's digests for this mesh (whole matrix at
    N=1, the rank's row block for N>1)."""
    try:
        data = json.loads(DIGESTS.read_text())
    except Exception:
        return {"checked": False, "why": "no digest file"}
    key = f"{config}/s{seed}" if world == 1 else f"{config}B/s{seed}/G{world}/b{rank}"
    ent = data.get(key)
    if ent is None:
        return {"checked": False, "why": f"no femasm digest for {key}"}
    if ent.get("mesh_sha256") and ent["mesh_sha256"] != mesh_sha:
        return {"checked": False, "why": "generated mesh differs from the digested one (numpy version?)"}
    got = csr_digests(rowptr, col[:nnz], val[:nnz])
    ok = (int(ent["nnz"]) == nnz and got[0] == ent["col_ptr_sha256"] and got[1] == ent["row_idx_sha256"]
          and got[2] == ent["values_sha256"])
    return {"checked": True, "match": bool(ok), "key": key, "nnz": nnz,
            "against": "SHA-256 of femasm OptV2 col_ptr/row_idx/values (tests/golden/reference_digests.json)"}


def mesh_sha256(sm):
    h = hashlib.sha256()
    for a in (sm.vertices.astype("<f8"), sm.connectivity.astype("<i8"), sm.weights.astype("<f8")):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


# ------------------------------------------------------------------------------------------
# our arm
# ------------------------------------------------------------------------------------------
def _allreduce(dist, t, op, gloo):
    if gloo:
        c = t.cpu()
        dist.all_reduce(c, op=op)
        return c.to(t.device)
    dist.all_reduce(t, op=op)
    return t


def dist_info(world):
    """Communicator facts for the JSON line (N > 1): backend, world size, NCCL version."""
    if world == 1:
        return None
    import torch
    import torch.distributed as dist

    info = {"backend": dist.get_backend(), "world_size": dist.get_world_size(), "rank_of_printer": dist.get_rank()}
    try:
        v = torch.cuda.nccl.version()
        info["nccl_version"] = ".".join(str(x) for x in v) if isinstance(v, tuple) else str(v)
    except Exception:  # noqa: BLE001 - informational only
        pass
    return info


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1305_3122_b200 as fa
    from paper_1305_3122_b200 import _lib
    from paper_1305_3122_b200.device import ResultBlock
    from paper_1305_3122_b200.dist import row_blocks
    from paper_1305_3122_b200.optv2 import HostAssembler

    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    # functional check of the N > 1 path on a single-GPU box (never a measurement):
    # FEMASM_BENCH_SAME_DEVICE=1 puts every rank on cuda:0, FEMASM_BENCH_BACKEND=gloo
    same_dev = os.environ.get("FEMASM_BENCH_SAME_DEVICE") == "1"
    gpu = 0 if same_dev else local
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    gloo = world > 1 and os.environ.get("FEMASM_BENCH_BACKEND", "nccl") == "gloo"
    if world > 1:
        backend = os.environ.get("FEMASM_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
        # the communicator every rank sees (stderr; the JSON line repeats it under "dist")
        print(f"[bench] rank {rank}/{world} backend={dist.get_backend()} world_size={dist.get_world_size()} "
              f"device=cuda:{gpu}", file=sys.stderr, flush=True)

    kind, n, lam, mu, sm = mesh_for(args.config, args.seed)
    me32 = np.ascontiguousarray(sm.connectivity, dtype=np.int32)
    me_d = torch.from_numpy(me32).to(dev)
    q_d = torch.from_numpy(sm.vertices).to(dev)
    w_d = torch.from_numpy(sm.weights).to(dev) if kind == "massw" else None
    # the mesh's areas, computed on the device with compute_areas' formula (mesh.py:51-69)
    a_d = torch.empty(sm.nme, dtype=torch.float64, device=dev)
    ar = ResultBlock()
    _lib.check(_lib.lib().fa_compute_areas(me_d.data_ptr(), sm.nme, q_d.data_ptr(), a_d.data_ptr(), ar.ptr,
                                           _lib.stream_handle()), "fa_compute_areas")
    q_use = q_d if kind in ("stiff", "elastic") else None
    # as assemble() does for a Mesh whose areas it computed: stiffness and elasticity recompute
    # them from the coordinates they gather anyway (bitwise compute_areas,
    # test_recomputed_areas_are_bitwise) instead of gathering one more array per incidence
    if kind in ("stiff", "elastic"):
        a_d = None
    v0, v1 = row_blocks(sm.nq, world)[rank]
    plan = fa.AssemblyPlan(sm.nme, sm.nq, v0, v1)
    plan.build(me_d)
    plan.check_build()
    n_rows = plan.rows(kind)
    cap = plan.capacity(kind)
    rowptr = torch.empty(n_rows + 1, dtype=torch.int64, device=dev)
    col = torch.empty(cap, dtype=torch.int32, device=dev)
    val = torch.empty(cap, dtype=torch.float64, device=dev)
    res = ResultBlock()
    nnz_t = torch.empty(world, dtype=torch.int64, device=dev)
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev)
    ev_rows0, ev_rows1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev_rows0.record(); ev_rows1.record()
    torch.cuda.synchronize()
    lib = _lib.lib()

    def compute(cold=True):
        # current stream (the capture stream inside a graph capture)
        if cold:  # fa_assemble_cold: plan build + numeric pass (weighted mass: W records in the build)
            plan.assemble_cold_into(me_d, kind, q_use, a_d, w_d, lam, mu, rowptr, col, val, res)
        else:
            plan.assemble_into(kind, q_use, a_d, w_d, lam, mu, rowptr, col, val, res)

    def exchange():
        if world > 1:
            if gloo:  # functional-check backend (CPU tensors)
                parts = [torch.empty(1, dtype=torch.int64) for _ in range(world)]
                dist.all_gather(parts, rowptr[-1:].cpu())
            else:
                dist.all_gather_into_tensor(nnz_t, rowptr[-1:])  # row-offset allgather (NCCL)

    def step(cold=True):
        compute(cold)
        exchange()

    # one cold (or warm) step captured as a CUDA graph: the launches of the ~9 kernels of a
    # step are replayed without host round trips (the kernel timer events are graph nodes)
    graphs = {}

    def graph_for(cold):
        if cold not in graphs:
            g = torch.cuda.CUDAGraph()
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                compute(cold)  # warm the capture stream
            torch.cuda.current_stream().wait_stream(side)
            torch.cuda.synchronize()
            lib.fa_set_kernel_timer(ev_rows0.cuda_event, ev_rows1.cuda_event)
            # thread-local capture: the NCCL watchdog thread's event queries stay legal
            with torch.cuda.graph(g, capture_error_mode="thread_local" if world > 1 else "global"):
                compute(cold)
            lib.fa_set_kernel_timer(None, None)
            torch.cuda.synchronize()
            graphs[cold] = g
        return graphs[cold]

    # the step's kernels replay as one CUDA graph at every N; for N > 1 the 8-byte NCCL nnz
    # allgather follows the replay eagerly on the same stream (gloo: functional checks only)
    use_graph = bool(args.graph) and not gloo

    def timed_loop(steps, cold):
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
        rows_ms = []
        g = graph_for(cold) if use_graph else None
        for i in range(steps):
            flush.zero_()
            starts[i].record()
            if g is not None:
                g.replay()
                exchange()
            else:
                lib.fa_set_kernel_timer(ev_rows0.cuda_event, ev_rows1.cuda_event)
                step(cold)
            ends[i].record()
            torch.cuda.synchronize()
            rows_ms.append(ev_rows0.elapsed_time(ev_rows1))
        lib.fa_set_kernel_timer(None, None)
        per = [s.elapsed_time(e) for s, e in zip(starts, ends)]
        return per, rows_ms

    for _ in range(args.warmup):
        step(True)
    torch.cuda.synchronize()
    clocks = ClockSampler(gpu)
    clocks.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.mark_start()
    per_step, rows_ms = timed_loop(args.steps, cold=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks.mark_end()
    clock_info = clocks.stop()
    r = res.fetch()
    rb = plan._build_res.fetch()
    local_nnz = int(r.nnz)
    total_ms = sum(per_step)
    # parity of what was timed: the last cold step's CSR against femasm's digests
    parity = {"checked": False, "why": "--verify 0"}
    if args.verify:
        parity = verify_output(args.config, args.seed, world, rank, rowptr, col, val, local_nnz, mesh_sha256(sm))
        parity["errors"] = {"degenerate_index": None if r.degenerate_index == _lib.INT64_MAX else int(r.degenerate_index),
                            "index_error_pos": None if rb.index_error_pos == _lib.INT64_MAX else int(rb.index_error_pos)}
    # warm: the plan reused (symbolic pattern reuse)
    warm_step, warm_rows = timed_loop(max(3, args.steps // 2), cold=False)
    warm_ms = sum(warm_step) / len(warm_step)
    t = torch.tensor([total_ms, warm_ms, float(np.mean(rows_ms))], dtype=torch.float64, device=dev)
    if world > 1:
        t = _allreduce(dist, t, dist.ReduceOp.MAX, gloo)
        nz = torch.tensor([local_nnz], dtype=torch.int64, device=dev)
        nz = _allreduce(dist, nz, dist.ReduceOp.SUM, gloo)
        total_nnz = int(nz.item())
    else:
        total_nnz = local_nnz
    total_ms, warm_ms, rows_avg_ms = (float(x) for x in t.tolist())
    value = sm.nme * args.steps / (total_ms * 1e-3)
    del flush
    torch.cuda.empty_cache()

    # end to end through the host-buffer API: pinned inputs -> device, plan, assemble, CSR -> host
    e2e = None
    if args.e2e_steps > 0:
        del col, val
        plan.close()
        torch.cuda.empty_cache()
        recompute = kind in ("stiff", "elastic")  # areas from q on the device, as above
        ha = HostAssembler(kind, sm.nq, sm.nme, v0, v1, recompute_areas=recompute, depth=2)
        pin = lambda x: torch.from_numpy(np.ascontiguousarray(x)).pin_memory()  # noqa: E731
        h_me = pin(me32)
        h_q = pin(sm.vertices) if kind in ("stiff", "elastic") else None
        h_a = None
        if not recompute:
            h_a = torch.empty(sm.nme, dtype=torch.float64).pin_memory()
            h_a.copy_(torch.from_numpy(fa.compute_areas(sm.vertices, sm.connectivity)))
        h_w = pin(sm.weights) if kind == "massw" else None
        lat = []
        for i in range(2 + 2):  # one warm-up per slot (pinned host buffers), then single synchronous calls
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            ha.run(h_me, h_q, h_a, h_w, lam, mu)
            if i >= 2:
                lat.append(time.perf_counter() - t0)
        # throughput: a stream of steps through submit/result over two slots; every step copies
        # its inputs in and its CSR out inside the timed region
        d2h = 0
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        prev = None
        for _ in range(args.e2e_steps):
            tk = ha.submit(h_me, h_q, h_a, h_w, lam, mu)
            if prev is not None:
                rp, cc, vv, nnz_e = ha.result(prev)
                d2h = rp.numel() * 8 + nnz_e * (4 + 8)
            prev = tk
        rp, cc, vv, nnz_e = ha.result(prev)
        d2h = rp.numel() * 8 + nnz_e * (4 + 8)
        t_stream = (time.perf_counter() - t0) / args.e2e_steps
        te = torch.tensor([t_stream, statistics.median(lat)], dtype=torch.float64, device=dev)
        if world > 1:
            te = _allreduce(dist, te, dist.ReduceOp.MAX, gloo)
        h2d = ha.bytes_h2d() * world
        d2h_t = torch.tensor([d2h], dtype=torch.int64, device=dev)
        if world > 1:
            d2h_t = _allreduce(dist, d2h_t, dist.ReduceOp.SUM, gloo)
        e2e = {"value": sm.nme / float(te[0]), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h_t.item()),
               "timing": f"wall clock over {args.e2e_steps} pipelined steps (submit/result, 2 slots), max over ranks",
               "latency_ms": float(te[1]) * 1e3, "latency": "one synchronous run() call, median of 2",
               "api": "paper_1305_3122_b200.optv2.HostAssembler.submit/result (C ABI fa_plan_build + fa_assemble)",
               "floor": "PCIe: the per-step D2H of the CSR bounds this (~55 GB/s measured, DESIGN.md §6)"}

    peak, peak_src = measured_peak()
    ab_rank = alg_bytes(kind, sm.nme, sm.nq, n_rows, local_nnz)
    achieved = ab_rank / (rows_avg_ms * 1e-3) / 1e9
    traffic = ncu_traffic(args.config) if world == 1 else None
    ab_total = alg_bytes(kind, sm.nme, sm.nq, (sm.nq * (2 if kind == "elastic" else 1)), total_nnz)
    cpu = None
    if rank == 0 and world == 1 and args.cpu_baseline_runs > 0:
        cpu = cpu_baseline(args.config, kind, sm, lam, mu, args.cpu_baseline_runs)

    if rank == 0:
        steps_list = launches_per_step(kind, sm.nme, sm.nq, v1 - v0)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": f"synthetic: seeded jittered/permuted unit-square mesh (SURVEY.md §8(d)), seed {args.seed}",
            "config": common_config(args.config, args.seed, sm),
            "nnz": total_nnz,
            "parallelism": f"row-blocks x{world}" if world > 1 else "single GPU",
            "step": "cold: plan build (part histogram, placement, per-part vertex sort) + fused row kernel "
                    "(+ NCCL nnz allgather when N>1), from device-resident me/q",
            "launch": ("CUDA graph replay per step" + (" + eager NCCL nnz allgather" if world > 1 else ""))
                      if use_graph else "eager launches",
            "dist": dist_info(world),
            "parity": parity,
            "hbm_gbs_whole_step": ab_total / (total_ms / args.steps * 1e-3) / 1e9,
            "roofline": {"bound": "hbm", "kernel": "k_rows (fused element + sparse() row kernel)",
                         "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic, "alg_bytes_per_launch": ab_rank, "avg_launch_ms": rows_avg_ms,
                         "peak_source": peak_src,
                         "alg_bytes": "12 B/tri me + 8 B/tri areas + 16 B/vertex q (stiff/elastic) or 8 B/vertex w "
                                      "(massw) + 8 B/row rowptr + 12 B/entry (col int32 + val f64); SURVEY.md §8(d)"},
            "roofline_whole_step_frac": (ab_total / (total_ms / args.steps * 1e-3) / 1e9) / peak,
            "warm": {"value": sm.nme / (warm_ms * 1e-3), "ms_per_step": warm_ms,
                     "what": "plan reused (vertex-sorted incidences cached): row kernel only"},
            "clocks": clock_info,
            "e2e": e2e,
            "gpu_launches": len(steps_list) * args.steps,
            "gpu_launches_detail": "per step: " + ", ".join(steps_list),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0 if (not parity.get("checked") or parity.get("match")) else 3


def main():
    args = parse_args()
    if args.config.upper() not in DESCR:
        raise SystemExit(f"unknown config {args.config}")
    args.config = args.config.upper()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
