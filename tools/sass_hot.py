"""Top stall-sampled SASS lines of one kernel from an ncu report: sass_hot.py REP KERNEL_REGEX [N]"""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{kern}", "-c", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
S = h.index("Warp Stall Sampling (All Samples)")
body = [r for r in rows[2:] if len(r) == len(h)]
def f(x):
    try: return float(x)
    except ValueError: return 0.0
tot = sum(f(r[S]) for r in body)
print("total samples", tot, "instructions", len(body))
for i, r in enumerate(body):
    r.append(i)
for r in sorted(body, key=lambda r: -f(r[S]))[:n]:
    print(f"{f(r[S]) / tot * 100:5.1f}%  #{r[-1]:5d} {r[1].strip()[:100]}")
