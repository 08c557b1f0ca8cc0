"""Per-kernel top warp stall reasons (cycles per issued instruction) from an ncu report."""
import csv, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
for v in rows[2:]:
    name = v[h.index("Kernel Name")][:40]
    st = [(c.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""), float(v[i] or 0))
          for i, c in enumerate(h) if c.startswith("smsp__average_warps_issue_stalled_") and c.endswith("_per_issue_active.ratio")]
    st.sort(key=lambda x: -x[1])
    print(name, " ".join(f"{a}={b:.1f}" for a, b in st[:8]))
