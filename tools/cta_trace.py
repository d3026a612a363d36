"""Summarise a CTA phase trace (ETD_CTA_TRACE=<stage> ETD_CTA_TRACE_OUT=file; the plan
writes it when it is destroyed): per-CTA fill / main-loop / epilogue cycles of the
fused backward launches on SMs 0-3, the phase offset of the two co-resident CTAs, and
the k-tile time with the partner CTA inside its main loop (shared) or outside (alone).

python tools/cta_trace.py TRACE.bin"""
import sys

import numpy as np

REC = 24
a = np.fromfile(sys.argv[1], dtype=np.uint64)
cnt = int(min(a[0], 8192))
r = a[8:8 + cnt * REC].reshape(cnt, REC).astype(np.int64)
print(f"{cnt} records")
for sm in range(4):
    x = r[r[:, 0] == sm]
    if len(x) < 50:
        continue
    x = x[np.argsort(x[:, 2])]
    brk = np.where(np.diff(x[:, 2]) > 2_000_000)[0]
    x = x[:(brk[0] + 1) if len(brk) else len(x)]
    t0, t1, t2, t3 = x[:, 2], x[:, 3], x[:, 4], x[:, 5]
    kt_end = x[:, 6:22]
    fill, main, epi = t1 - t0, t2 - t1, t3 - t2
    span = t3.max() - t0.min()
    gaps = np.diff(t0)
    print(f"SM {sm}: {len(x)} CTAs over {span} cycles; fill {np.median(fill):.0f}, main {np.median(main):.0f}, "
          f"epilogue {np.median(epi):.0f}; start-to-start {np.median(gaps):.0f} (p10 {np.percentile(gaps, 10):.0f}, "
          f"p90 {np.percentile(gaps, 90):.0f})")
    # k-tile durations classified by the partner's state over the k-tile
    shared, alone, mixed = [], [], []
    for i in range(2, len(x) - 2):
        starts = np.concatenate(([t1[i]], kt_end[i, :-1]))
        for k in range(16):
            lo, hi = starts[k], kt_end[i, k]
            if hi <= lo:
                continue
            ov = 0
            for j in (i - 2, i - 1, i + 1, i + 2):
                ov += max(0, min(hi, t2[j]) - max(lo, t1[j]))
            frac = ov / (hi - lo)
            (shared if frac > 0.98 else alone if frac < 0.02 else mixed).append(hi - lo)
    for name, v in (("shared", shared), ("alone", alone), ("mixed", mixed)):
        if v:
            v = np.array(v)
            print(f"   k-tile {name}: n={len(v)} median {np.median(v):.0f} mean {v.mean():.0f} p10 {np.percentile(v, 10):.0f} "
                  f"p90 {np.percentile(v, 90):.0f}")
