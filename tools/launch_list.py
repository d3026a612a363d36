"""Markdown launch list from an `ncu --metrics gpu__time_duration.sum --csv --log-file` capture.
python tools/launch_list.py LAUNCHES.csv OUT.md "command that was profiled" """
import csv
import io
import sys

src, out, cmd = sys.argv[1], sys.argv[2], sys.argv[3]
lines = [l for l in open(src).read().splitlines() if l.startswith('"')]
rows = list(csv.reader(io.StringIO("\n".join(lines))))
h = rows[0]
K, G, V, U = h.index("Kernel Name"), h.index("Grid Size"), h.index("Metric Value"), h.index("Metric Unit")
recs = []
for r in rows[1:]:
    ms = float(r[V].replace(",", "")) * {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "msecond": 1.0, "ms": 1.0}.get(r[U], 1e-6)
    recs.append((r[K].split("(")[0].replace("void ", ""), r[G], ms))
tot = sum(x[2] for x in recs)
with open(out, "w") as f:
    f.write(f"# Launch list — `{cmd}`\n\n")
    f.write("`ncu --metrics gpu__time_duration.sum --clock-control none` (serialised, cold-cache; compare shares).\n\n")
    f.write(f"{len(recs)} launches, {tot:.1f} ms in total.\n\n| # | kernel | grid | ms | share |\n|---|---|---|---|---|\n")
    for i, (k, g, ms) in enumerate(recs):
        f.write(f"| {i} | `{k}` | {g} | {ms:.3f} | {100 * ms / tot:.1f}% |\n")
print(len(recs), tot)
