#!/usr/bin/env python
"""Benchmark of the B200 OptV2 P1 assembly (one JSON line on rank 0).

Metric (BASELINE.json): triangles assembled per second, device-timed, including the CSR
build, plus achieved HBM GB/s.  Workload: BASELINE configs[1] = C2, the P1 weighted mass
matrix on the seeded jittered/permuted unit-square mesh with N=1024 (2,097,152 triangles,
1,050,625 vertices, vertex weights U(0.5, 2)); other configs via --config.

One step = one complete OptV2 assembly from device-resident inputs: plan build (part
histogram, staged part placement, per-part vertex sort) + fused row kernel writing
rowptr/col/val, i.e. the reference's `assemble(mesh, kind, OPTV2)` with nothing cached between
steps ("cold").  The L2
is flushed (a 512 MB buffer is zeroed) between timed steps, outside the timed windows.
N > 1 (torchrun): rank g assembles the matrix rows of vertex block g (row-block
decomposition); the step includes the NCCL allgather of the per-rank nnz
that yields the global row offsets.  The total work is fixed: "scaling": "strong".

--impl reference: the reference algorithm on the host CPU (the numpy restatement of femasm's
OptV2 in oracle/, femasm itself being pure Python/numpy and not shippable), run on all host
cores as one row-block subset per process.  Rank 0 only.
"""

from __future__ import annotations

import argparse
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
def launches_per_step(kind, nme, nq, nv):
    """Our kernels launched per cold step (fa_assemble_cold); memsets are not counted.  The
    two-level plan rule mirrors fa_plan_create (more than 8192 parts of 1024 rows, or more than
    160 MB of part records with more than 256 parts) and adds k_part_split."""
    nparts = -(-nv // 1024)
    two_level = nparts > 8192 or (48 * nme // max(nq, 1) * nv > (160 << 20) and nparts > 256)
    hist = "k_part_hist (weighted mass: also the per-triangle W records)" if kind == "massw" else "k_part_hist"
    return (["k_reset", hist, "k_part_scan", "k_part_place"] + (["k_part_split"] if two_level else [])
            + ["k_part_sort", "k_reset", "k_rows", "k_compact (exits at once unless a sum was exactly zero)"])
DEFAULT_CONFIG = "C2"
DESCR = {
    "C1": "P1 mass, N=256 seeded jittered/permuted unit square",
    "C2": "P1 weighted mass (vertex weights U(0.5,2)), N=1024 seeded jittered/permuted unit square",
    "C3": "P1 stiffness, N=2048 seeded jittered/permuted unit square",
    "C4": "2D linear elasticity lam=1 mu=0.5, N=2048 seeded jittered/permuted unit square",
    "C5": "P1 stiffness, N=8192 seeded jittered/permuted unit square",
}


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default=DEFAULT_CONFIG)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--cpu-baseline-runs", type=int, default=2, help="timed runs of the 1-core CPU baseline (0: skip)")
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--graph", type=int, default=1, help="replay each step as a captured CUDA graph (N=1)")
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


def alg_bytes(kind, nme, nq, n_rows, nnz, owned_all=True):
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

    A background thread issues single-shot queries back to back (a looping nvidia-smi writing
    into a pipe buffers its output and loses it when terminated); every sample is timestamped
    and the summary keeps the samples taken inside [mark_start, mark_end].  When the timed region
    is shorter than one query, the samples adjacent to it are reported and flagged."""

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
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
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


def cpu_baseline_port(kind, sm, lam, mu, runs):
    """1-core CPU baseline: the numpy restatement of femasm's OptV2 (oracle/), timed like
    femasm bench._time_cell (one discarded warm-up, median of the timed runs)."""
    from oracle import femasm_oracle as fo

    areas = fo.triangle_areas(sm.vertices, sm.connectivity)
    times = []
    for i in range(runs + 1):
        t0 = time.perf_counter()
        fo.assemble_optv2(kind, sm.vertices, sm.connectivity, areas, sm.weights, lam, mu)
        dt = time.perf_counter() - t0
        if i > 0:
            times.append(dt)
    t = statistics.median(times)
    return {"value": sm.nme / t, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"full mesh ({sm.nme} triangles), numpy OptV2 restatement, median of {runs} after 1 warm-up",
            "seconds_per_assembly": t}


# ------------------------------------------------------------------------------------------
# reference arm: the reference algorithm on every host core (row-block subsets in processes)
# ------------------------------------------------------------------------------------------
_REF = {}


def _ref_block(args):
    from oracle import femasm_oracle as fo

    v0, v1 = args
    d = _REF
    ptr, idx, vals = fo.assemble_row_block(d["kind"], d["V"], d["C"], d["areas"], d["w"], d["lam"], d["mu"], v0, v1)
    return int(ptr[-1])


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    import multiprocessing as mp

    from oracle import femasm_oracle as fo
    from paper_1305_3122_b200.dist import row_blocks

    kind, n, lam, mu, sm = mesh_for(args.config, args.seed)
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    _REF.update(kind=kind, V=sm.vertices, C=sm.connectivity, areas=fo.triangle_areas(sm.vertices, sm.connectivity),
                w=sm.weights, lam=lam, mu=mu)
    blocks = row_blocks(sm.nq, cores)
    ctx = mp.get_context("fork")
    times = []
    with ctx.Pool(cores) as pool:
        for i in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            nnz = sum(pool.map(_ref_block, blocks))
            dt = time.perf_counter() - t0
            if i >= args.warmup:
                times.append(dt)
    total = sum(times)
    value = sm.nme * len(times) / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total / len(times) * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic: seeded jittered/permuted unit-square mesh (SURVEY.md §8(d)), seed {args.seed}",
        "config": {"workload": f"{args.config}: {DESCR[args.config]}", "nq": sm.nq, "nme": sm.nme, "nnz": nnz,
                   "seed": args.seed, "parallelism": f"{cores} host processes x row-block subset"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"full mesh per step as {cores} row-block subsets (femasm OptV2 numpy restatement)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


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

    kind, n, lam, mu, sm = mesh_for(args.config, args.seed)
    areas = fa.compute_areas(sm.vertices, sm.connectivity)
    me32 = np.ascontiguousarray(sm.connectivity, dtype=np.int32)
    me_d = torch.from_numpy(me32).to(dev)
    q_d = torch.from_numpy(sm.vertices).to(dev)
    a_d = torch.from_numpy(areas).to(dev)
    w_d = torch.from_numpy(sm.weights).to(dev) if kind == "massw" else None
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
    stream = torch.cuda.current_stream()
    ev_rows0, ev_rows1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev_rows0.record(); ev_rows1.record()
    torch.cuda.synchronize()
    lib = _lib.lib()

    def step(cold=True):
        # current stream (the capture stream inside a graph capture)
        if cold:  # fa_assemble_cold: plan build + numeric pass (weighted mass: W records in the build)
            plan.assemble_cold_into(me_d, kind, q_use, a_d, w_d, lam, mu, rowptr, col, val, res)
        else:
            plan.assemble_into(kind, q_use, a_d, w_d, lam, mu, rowptr, col, val, res)
        if world > 1:
            if gloo:  # functional-check backend (CPU tensors)
                parts = [torch.empty(1, dtype=torch.int64) for _ in range(world)]
                dist.all_gather(parts, rowptr[-1:].cpu())
            else:
                dist.all_gather_into_tensor(nnz_t, rowptr[-1:])  # row-offset allgather (NCCL)

    # one cold (or warm) step captured as a CUDA graph: the launches of the ~8 kernels of a
    # step are replayed without host round trips (the kernel timer events are graph nodes)
    graphs = {}

    def graph_for(cold):
        if cold not in graphs:
            g = torch.cuda.CUDAGraph()
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                step(cold)  # warm the capture stream
            torch.cuda.current_stream().wait_stream(side)
            torch.cuda.synchronize()
            lib.fa_set_kernel_timer(ctypes_ptr(ev_rows0), ctypes_ptr(ev_rows1))
            with torch.cuda.graph(g):
                step(cold)
            lib.fa_set_kernel_timer(None, None)
            torch.cuda.synchronize()
            graphs[cold] = g
        return graphs[cold]

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
            else:
                lib.fa_set_kernel_timer(ctypes_ptr(ev_rows0), ctypes_ptr(ev_rows1))
                step(cold)
            ends[i].record()
            torch.cuda.synchronize()
            rows_ms.append(ev_rows0.elapsed_time(ev_rows1))
        lib.fa_set_kernel_timer(None, None)
        per = [s.elapsed_time(e) for s, e in zip(starts, ends)]
        return per, rows_ms

    def ctypes_ptr(ev):
        return ev.cuda_event

    use_graph = args.graph and world == 1  # (NCCL collectives stay eager for N > 1)

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
    local_nnz = int(r.nnz)
    total_ms = sum(per_step)
    # warm: the plan reused (symbolic pattern reuse)
    warm_step, _ = timed_loop(max(3, args.steps // 2), cold=False)
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

    # end to end through the host-buffer API: pinned inputs -> device, plan, assemble, CSR -> host
    e2e = None
    if args.e2e_steps > 0:
        recompute = kind in ("stiff", "elastic")  # areas from q on the device, as above
        ha = HostAssembler(kind, sm.nq, sm.nme, v0, v1, recompute_areas=recompute, depth=2)
        pin = lambda x: torch.from_numpy(np.ascontiguousarray(x)).pin_memory()  # noqa: E731
        h_me, h_q, h_a = pin(me32), pin(sm.vertices), (None if recompute else pin(areas))
        h_w = pin(sm.weights) if kind == "massw" else None
        h_q = h_q if kind in ("stiff", "elastic") else None
        lat = []
        for i in range(2 + 3):  # warm-up, then the latency of single synchronous calls
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
               "latency_ms": float(te[1]) * 1e3, "latency": "one synchronous run() call, median of 3",
               "api": "paper_1305_3122_b200.optv2.HostAssembler.submit/result (C ABI fa_plan_build + fa_assemble)"}

    peak, peak_src = measured_peak()
    ab_rank = alg_bytes(kind, sm.nme, sm.nq, n_rows, local_nnz)
    achieved = ab_rank / (rows_avg_ms * 1e-3) / 1e9
    traffic = ncu_traffic(args.config) if world == 1 else None
    ab_total = alg_bytes(kind, sm.nme, sm.nq, (sm.nq * (2 if kind == "elastic" else 1)), total_nnz)
    cpu = None
    if rank == 0 and world == 1 and args.cpu_baseline_runs > 0:
        cpu = cpu_baseline_port(kind, sm, lam, mu, args.cpu_baseline_runs)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": f"synthetic: seeded jittered/permuted unit-square mesh (SURVEY.md §8(d)), seed {args.seed}",
            "config": {"workload": f"{args.config}: {DESCR[args.config]}", "nq": sm.nq, "nme": sm.nme, "nnz": total_nnz,
                       "seed": args.seed, "parallelism": f"row-blocks x{world}" if world > 1 else "single GPU",
                       "step": "cold: plan build (part histogram, placement, per-part vertex sort) + fused row "
                               "kernel (+ NCCL nnz allgather when N>1)",
                       "l2": "512 MB buffer zeroed between timed steps (outside the timed windows)",
                       "launch": "CUDA graph replay per step" if (args.graph and world == 1) else "eager launches"},
            "hbm_gbs_whole_step": ab_total / (total_ms / args.steps * 1e-3) / 1e9,
            "roofline": {"bound": "hbm", "kernel": "k_rows (fused element + sparse() row kernel)",
                         "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic, "alg_bytes_per_launch": ab_rank, "avg_launch_ms": rows_avg_ms,
                         "peak_source": peak_src},
            "roofline_whole_step_frac": (ab_total / (total_ms / args.steps * 1e-3) / 1e9) / peak,
            "warm": {"value": sm.nme / (warm_ms * 1e-3), "ms_per_step": warm_ms,
                     "what": "plan reused (vertex-sorted incidences cached): row kernel only"},
            "clocks": clock_info,
            "e2e": e2e,
            "gpu_launches": len(launches_per_step(kind, sm.nme, sm.nq, v1 - v0)) * args.steps,
            "gpu_launches_detail": "per step: " + ", ".join(launches_per_step(kind, sm.nme, sm.nq, v1 - v0)),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


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
