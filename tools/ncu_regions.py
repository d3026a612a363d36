"""Split one kernel's per-SASS-instruction stall samples (ncu source page, CSV) into
prologue / main loop / epilogue and report the stall reasons of each region.
The main loop is the address range from the first to the last DMMA.
python tools/ncu_regions.py SOURCE.csv [more.csv ...]"""
import csv
import sys

REASONS = ["stall_barrier", "stall_branch_resolving", "stall_dispatch", "stall_drain", "stall_lg", "stall_long_sb",
           "stall_math", "stall_membar", "stall_mio", "stall_misc", "stall_no_inst", "stall_not_selected",
           "stall_selected", "stall_short_sb", "stall_sleep", "stall_tex", "stall_wait"]


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


def analyse(path):
    rows = list(csv.reader(open(path)))
    name, h = rows[0][1], rows[1]
    data = []
    for r in rows[2:]:
        if not r or r[0] in ("Kernel Name", "Address"):
            break
        data.append(r)
    col = {k: h.index(k) for k in ["Source", "Warp Stall Sampling (All Samples)", "Instructions Executed"] + REASONS}
    dm = [i for i, r in enumerate(data) if "DMMA" in r[col["Source"]]]
    lo, hi = dm[0], dm[-1]
    regions = {"prologue": data[:lo], "main loop": data[lo:hi + 1], "epilogue": data[hi + 1:]}
    tot = sum(f(r[col["Warp Stall Sampling (All Samples)"]]) for r in data) or 1.0
    out = [f"kernel: {name[:150]}", f"instructions: {len(data)}; DMMA instructions in the SASS: {len(dm)}"]
    for reg, rs in regions.items():
        s = sum(f(r[col["Warp Stall Sampling (All Samples)"]]) for r in rs)
        ins = sum(f(r[col["Instructions Executed"]]) for r in rs)
        rs_sum = {k: sum(f(r[col[k]]) for r in rs) for k in REASONS}
        top = sorted(rs_sum.items(), key=lambda x: -x[1])[:6]
        out.append(f"  {reg:10s} samples {s / tot * 100:5.1f}%  warp-instr {ins:.3e}  top: " +
                   ", ".join(f"{k[6:]} {v / tot * 100:.1f}%" for k, v in top if v > 0))
    return "\n".join(out)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(analyse(p))
