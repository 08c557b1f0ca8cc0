"""Duration, instructions, IPC and stall cycles per issued instruction of the first kernel in
ncu reports: ncu_stalls2.py REP [REP...]"""
import csv, subprocess, sys
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    d = dict(zip(rows[0], rows[2]))
    st = []
    for a, b in d.items():
        if a.startswith("smsp__average_warps_issue_stalled_") and a.endswith("_per_issue_active.ratio"):
            try:
                x = float(b)
            except ValueError:
                continue
            if x > 0.05:
                st.append((x, a.split("stalled_")[1].replace("_per_issue_active.ratio", "")))
    print(f"{rep}: {d.get('Kernel Name', '')[:30]} t={d['gpu__time_duration.sum']}us inst={d['smsp__inst_executed.sum']} "
          f"ipc={float(d['sm__inst_executed.avg.per_cycle_active']):.2f}")
    print("   " + " ".join(f"{n}={x:.2f}" for x, n in sorted(st, reverse=True)))
