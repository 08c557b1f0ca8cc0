"""Attribute ncu per-SASS instruction counts / stall samples to source lines via nvdisasm -gi.
usage: sass_lines.py REP KERNEL_REGEX MANGLED_FUNC [SO]"""
import csv, re, subprocess, sys, tempfile, os, collections
rep, kre, func = sys.argv[1:4]
so = sys.argv[4] if len(sys.argv) > 4 else "paper_1305_3122_b200/libfemasm_b200.so"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{kre}", "-c", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
E, S = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
body = [r for r in rows[2:] if len(r) == len(h)]
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=d, capture_output=True)
cub = [f for f in os.listdir(d) if f.startswith("fa_assembly")][0]
asm = subprocess.run(["nvdisasm", "-gi", "-c", os.path.join(d, cub)], capture_output=True, text=True).stdout
lines = asm.splitlines()
start = lines.index(f"{func}:")
chain, seq, inner, outer = [], [], None, None
for line in lines[start + 1:]:
    if line.startswith(".text.") or line.startswith("//----"):
        if seq: break
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', line)
    if m:
        chain.append(f"{os.path.basename(m.group(1))}:{m.group(2)}")
        continue
    if re.match(r"\s+/\*[0-9a-f]{4,}\*/", line):
        if chain:
            inner = chain[0]
            outs = [c for c in chain if c.startswith("fa_assembly.cu")]
            outer = outs[-1] if outs else chain[-1]
            chain = []
        seq.append(f"{outer} [{inner}]" if inner != outer else outer)
print("ncu instrs", len(body), "disasm instrs", len(seq))
n = min(len(body), len(seq))
f = lambda x: float(x) if x not in ("", None) else 0.0
agg, aggf = collections.Counter(), collections.Counter()
stl, stlf = collections.Counter(), collections.Counter()
for i in range(n):
    e, s = f(body[i][E]), f(body[i][S])
    agg[seq[i]] += e; stl[seq[i]] += s
    key = (seq[i] or "?").split("[")[-1].split(":")[0]
    aggf[key] += e; stlf[key] += s
te, ts = sum(agg.values()), sum(stl.values())
if os.environ.get("PHASES"):  # "name:lo-hi,name:lo-hi" line ranges of the kernel file (outer line)
    ph = [(nm, int(r.split("-")[0]), int(r.split("-")[1])) for nm, r in (x.split(":") for x in os.environ["PHASES"].split(","))]
    pe, ps = collections.Counter(), collections.Counter()
    for k in agg:
        try:
            ln = int(k.split(" ")[0].split(":")[1])
        except (IndexError, ValueError):
            ln = -1
        nm = next((n for n, lo, hi in ph if lo <= ln <= hi), "other")
        pe[nm] += agg[k]; ps[nm] += stl[k]
    print("by phase:", {k: f"{v/te*100:.1f}% inst / {ps[k]/ts*100:.1f}% stall" for k, v in pe.most_common()})
print("by file:", {k: f"{v/te*100:.1f}%/{stlf[k]/ts*100:.1f}%" for k, v in aggf.most_common()})
for k, v in agg.most_common(int(os.environ.get("TOP", 40))):
    print(f"{v/te*100:5.1f}% inst {stl[k]/ts*100:5.1f}% stall  {k}")
