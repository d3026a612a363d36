"""Per-stage time of every tile class on the small BASELINE configs (dev tool).

python tools/tile_sweep.py [cfg ids...]   -> one line per (config, stage): ms per tile class
Each class is forced with ETD_FORCE_TILE in a fresh subprocess; '-' = the heuristic.
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(cfg, tile):
    env = dict(os.environ)
    env.pop("ETD_FORCE_TILE", None)
    if tile != "-":
        env["ETD_FORCE_TILE"] = tile
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "quick_perf.py"), str(cfg), "--steps", "5"],
                         capture_output=True, text=True, env=env).stdout.strip().splitlines()
    rec = json.loads(out[-1])
    return rec["ms_per_step"], {s["name"]: s["ms"] for s in rec["stages"]}


if __name__ == "__main__":
    for cfg in [int(a) for a in sys.argv[1:]] or [1, 2]:
        res = {t: run(cfg, t) for t in ["-", "0", "1", "2", "3"]}
        print(f"config {cfg}: ms/step " + " ".join(f"{t}:{res[t][0]:.4f}" for t in res))
        for st in res["-"][1]:
            print(f"  {st:12s} " + " ".join(f"{t}:{res[t][1].get(st, float('nan')):.4f}" for t in res))
