"""Parity-split (FOLD) vs dense transforms on small grids (dev tool).

python tools/fold_debug.py            -> runs every case in a subprocess
python tools/fold_debug.py dim n axes -> one case (ETD_FOLD_AXES = axes)
"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402


def case(dim, n, axes):
    import paper_2601_06849_b200 as etd

    def plan(dense):
        os.environ["ETD_DENSE"] = "1" if dense else "0"
        os.environ["ETD_FOLD_AXES"] = str(axes)
        return etd.make_plan(etd.unit_box_grid(dim, n + 1), 0.01, 1.0, 1.0, source=etd.allen_cahn_cubic())

    rng = np.random.default_rng(1)
    x = rng.standard_normal(n ** dim)
    pf, pd = plan(False), plan(True)
    for axis in range(dim):
        a, b = pf.apply_Q(1, x, axis), pd.apply_Q(1, x, axis)
        print(f"dim {dim} n {n} axes {axes} axis {axis} apply_Q max|fold-dense| {np.abs(a - b).max():.3e}", flush=True)
    u = 0.5 * np.sin(np.linspace(0, 3, n ** dim))
    ra = etd.advance(pf, etd.StepperState(0, 0.0, u), etd.allen_cahn_cubic(), nsteps=2)
    rb = etd.advance(pd, etd.StepperState(0, 0.0, u), etd.allen_cahn_cubic(), nsteps=2)
    print(f"dim {dim} n {n} axes {axes} step gap {np.abs(ra.U - rb.U).max():.3e}", flush=True)


if __name__ == "__main__":
    if len(sys.argv) == 4:
        case(*[int(a) for a in sys.argv[1:]])
    else:
        for dim, n, axes in [(2, 15, 1), (2, 16, 1), (2, 15, 3), (2, 127, 3), (3, 15, 7), (3, 31, 7), (3, 32, 7), (3, 47, 7)]:
            r = subprocess.run([sys.executable, __file__, str(dim), str(n), str(axes)], capture_output=True, text=True)
            print(r.stdout.strip() or f"dim {dim} n {n} axes {axes}: FAILED {r.stderr.strip().splitlines()[-1][:200]}",
                  flush=True)
