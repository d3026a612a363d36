"""Thomas-backend smoke over sizes (dev tool): two steps of a scalar plan per size.
python tools/thomas_dbg.py DIM N [N ...]"""
import os
import sys, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_06849_b200 as etd
dim = int(sys.argv[1]); sizes = [int(x) for x in sys.argv[2:]]
for n in sizes:
    g = etd.unit_box_grid(dim, n + 1)
    u0 = np.random.default_rng(1).uniform(-1, 1, n ** dim)
    try:
        p = etd.make_plan(g, 5e-4, 0.5, 0.0, backend=etd.BackendKind.Thomas)
        out = etd.advance(p, etd.StepperState(0, 0.0, u0), etd.allen_cahn_cubic(), nsteps=2)
        print(n, "ok", float(np.max(np.abs(out.U))), flush=True)
    except Exception as e:
        print(n, "FAIL", e, flush=True)
        break
