"""Summarise an ncu --set full report of etd_contract launches into profiles/.

python tools/ncu_summary.py REPORT.ncu-rep STAGE_NAMES(comma) OUT.md [traffic_key]
Writes a markdown table and merges per-stage DRAM bytes into profiles/ncu_traffic.json
under traffic_key (e.g. cfg4_n1023) for bench.py's roofline.traffic.
"""
import csv
import io
import json
import os
import subprocess
import sys

WANT = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "dmma_pct"),
    ("sm__inst_executed_pipe_tensor_subpipe_dmma.sum", "dmma_inst"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "lds_conflicts"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall_wait"),
    ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", "stall_pipe"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall_barrier"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall_long_sb"),
]
SCALE = {"ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main():
    rep, names, out = sys.argv[1], sys.argv[2].split(","), sys.argv[3]
    key = sys.argv[4] if len(sys.argv) > 4 else None
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    recs = []
    for i, r in enumerate(data):
        rec = {"stage": names[i] if i < len(names) else f"launch{i}", "kernel": r[hdr.index("Kernel Name")][:60]}
        for m, k in WANT:
            if m in hdr:
                j = hdr.index(m)
                try:
                    v = float(r[j].replace(",", ""))
                except ValueError:
                    continue
                if v != v:  # ncu could not collect (e.g. replay memory save/restore failed)
                    continue
                rec[k] = v * SCALE.get(units[j], 1.0) if k in ("time", "dram_read", "dram_write") else v
        recs.append(rec)
    lines = ["| stage | time ms | DRAM read GB | DRAM write GB | DMMA pipe % | DMMA inst | LDS bank conflicts | regs | "
             "stall wait | stall pipe | stall barrier |",
             "|---|---|---|---|---|---|---|---|---|---|---|"]
    def fmt(r, k, scale=1.0, spec=".2f"):
        return format(r[k] * scale, spec) if k in r else "n/a"

    for r in recs:
        lines.append("| " + " | ".join([r["stage"], fmt(r, "time", 1e3, ".3f"), fmt(r, "dram_read", 1e-9),
                                        fmt(r, "dram_write", 1e-9), fmt(r, "dmma_pct", 1, ".1f"),
                                        fmt(r, "dmma_inst", 1, ".3g"), fmt(r, "lds_conflicts", 1, ".0f"),
                                        fmt(r, "regs", 1, ".0f"), fmt(r, "stall_wait"), fmt(r, "stall_pipe"),
                                        fmt(r, "stall_barrier")]) + " |")
    with open(out, "w") as f:
        f.write(f"# ncu --set full summary: {os.path.basename(rep)}\n\n")
        f.write("Serialised, cold-cache replays (ncu): compare shares, not absolute step times.\n\n")
        f.write("\n".join(lines) + "\n")
        f.write("\nn/a: ncu could not replay that launch (device-memory save/restore of the ~103 GB working set);"
                " only the first captured launch has the full metric set.\n")
    if key:
        path = os.path.join(os.path.dirname(out), "ncu_traffic.json")
        db = json.load(open(path)) if os.path.exists(path) else {}
        db.setdefault(key, {}).update({r["stage"]: r["dram_read"] + r["dram_write"] for r in recs
                                        if "dram_read" in r and "dram_write" in r})
        json.dump(db, open(path, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
