"""Write profiles/<tag>_* summaries from ncu outputs in gpurun_out/.

usage: make_profile_summary.py TAG CONFIG LAUNCH_CSV FULL_REP [FULL_REP ...]
  - profiles/<tag>_launches_<config>.csv   (the gpu__time_duration launch list, verbatim)
  - profiles/<tag>_ncu_<config>.md          (per-kernel share + --set full metrics + stalls)
  - profiles/ncu_summary.json               (DRAM bytes per k_rows launch: bench.py roofline.traffic)
"""
import collections, csv, json, shutil, subprocess, sys
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
tag, cfg, launch_csv, reps = sys.argv[1], sys.argv[2], sys.argv[3], sys.argv[4:]
prof = REPO / "profiles"
prof.mkdir(exist_ok=True)
shutil.copy(launch_csv, prof / f"{tag}_launches_{cfg}.csv")

rows = [r for r in csv.reader(open(launch_csv)) if len(r) > 10]
h = rows[0]
K, V, U = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.OrderedDict()
for r in rows[1:]:
    nm = r[K].split("(")[0].replace("void ", "")
    v = float(r[V].replace(",", "")) * {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(r[U], 1e-3)
    agg.setdefault(nm, []).append(v)
ours = {k: v for k, v in agg.items() if k.startswith("fa::") and "k_areas" not in k and "reset_result_b" not in k}

M = {"gpu__time_duration.sum": "duration (us)", "dram__bytes_read.sum": "DRAM read (MB)",
     "dram__bytes_write.sum": "DRAM write (MB)", "lts__t_sector_hit_rate.pct": "L2 hit %",
     "sm__warps_active.avg.pct_of_peak_sustained_active": "warps active %",
     "smsp__inst_executed.sum": "warp instructions", "sm__inst_executed.avg.per_cycle_active": "IPC",
     "launch__registers_per_thread": "registers", "l1tex__t_sectors_pipe_lsu_mem_local_op_st.sum": "local st sectors"}
full = collections.OrderedDict()
stalls = {}
for rep in reps:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(out.splitlines()))
    hh, units = rr[0], rr[1]
    SCALE = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "Tbyte": 1e6,   # -> MB
             "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6,         # -> us
             "ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6}
    def conv(m, raw):
        u = units[hh.index(m)]
        try:
            x = float(raw.replace(",", ""))
        except ValueError:
            return raw
        return f"{x * SCALE.get(u, 1.0):.6g}" if u in SCALE else f"{x:.6g}"
    for v in rr[2:]:
        name = v[hh.index("Kernel Name")].split("(")[0].replace("void ", "")
        full[name] = {lab: conv(m, v[hh.index(m)]) for m, lab in M.items() if m in hh}
        st = [(c.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""), float(v[i] or 0))
              for i, c in enumerate(hh) if c.startswith("smsp__average_warps_issue_stalled_") and c.endswith("_per_issue_active.ratio")]
        stalls[name] = sorted(st, key=lambda x: -x[1])[:6]

tot = sum(sum(v) / len(v) for v in ours.values())
md = [f"# ncu summary, {tag}, config {cfg}", "",
      f"Commands (config {cfg}): launch list `ncu --metrics gpu__time_duration.sum --clock-control none -c 400 python bench.py --config {cfg} --steps 2 --warmup 1 --e2e-steps 0 --cpu-baseline-runs 0 --verify 0` (graph replay: the warm steps are in the list too);",
      f"full: `ncu --set full --import-source on --clock-control none -k regex:k_rows -c 1 python bench.py --config {cfg} --steps 1 --warmup 1 --e2e-steps 0 --cpu-baseline-runs 0 --verify 0 --graph 0` (bench mode: recomputed areas for stiffness/elasticity).",
      "Launch-list times are cold-cache and serialised: compare shares, not absolutes.", "",
      "## Per-step launch list (average over launches)", "", "| kernel | launches | avg us | share of step |", "|---|---|---|---|"]
for k, v in ours.items():
    a = sum(v) / len(v)
    md.append(f"| `{k}` | {len(v)} | {a:.1f} | {a / tot * 100:.1f}% |")
md += ["", f"Sum of our kernels per step: {tot:.1f} us", "", "## --set full", ""]
labs = list(M.values())
md.append("| kernel | " + " | ".join(labs) + " |")
md.append("|---" * (len(labs) + 1) + "|")
for k, d in full.items():
    md.append(f"| `{k}` | " + " | ".join(d.get(l, "") for l in labs) + " |")
md += ["", "## Top stall reasons (cycles per issued instruction)", ""]
for k, st in stalls.items():
    md.append(f"- `{k}`: " + ", ".join(f"{a} {b:.1f}" for a, b in st))
(prof / f"{tag}_ncu_{cfg}.md").write_text("\n".join(md) + "\n")

summ_p = prof / "ncu_summary.json"
summ = json.loads(summ_p.read_text()) if summ_p.exists() else {"configs": {}}
for k, d in full.items():
    if "k_rows" in k:
        summ["configs"].setdefault(cfg, {})["k_rows"] = {
            "dram_bytes_read": float(d["DRAM read (MB)"]) * 1e6, "dram_bytes_write": float(d["DRAM write (MB)"]) * 1e6,
            "duration_us": float(d["duration (us)"]), "source": f"profiles/{tag}_ncu_{cfg}.md", "tag": tag}
summ_p.write_text(json.dumps(summ, indent=1) + "\n")
print((prof / f"{tag}_ncu_{cfg}.md").read_text())
