"""Top SASS stall hotspots of the first kernel in an ncu report (text summary).
python tools/ncu_hotspots.py REPORT.ncu-rep OUT.txt"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep, out = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--launch-count", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[1]
data = []
for r in rows[2:]:
    if r and r[0] in ("Kernel Name", "Address"):
        break
    data.append(r)
si = h.index("Warp Stall Sampling (All Samples)")
tot = sum(float(r[si] or 0) for r in data) or 1.0
agg = defaultdict(float)
for r in data:
    op = r[1].split()[0] if r[1] else ""
    if op.startswith("@"):
        op = r[1].split()[1]
    agg[op.split(".")[0]] += float(r[si] or 0)
with open(out, "w") as f:
    f.write(f"kernel: {rows[0][1][:160]}\nstall samples by opcode (share of all samples):\n")
    for k, v in sorted(agg.items(), key=lambda x: -x[1])[:12]:
        f.write(f"  {k:12s} {v / tot * 100:5.1f}%\n")
    f.write("top instructions:\n")
    for r in sorted(data, key=lambda r: -float(r[si] or 0))[:15]:
        f.write(f"  {float(r[si]) / tot * 100:5.2f}%  {r[1][:90]}\n")
print(open(out).read())
