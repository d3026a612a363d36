"""GPU: the CUDA path (C-ABI) against the committed golden fixtures made by the
reference itself (tests/golden/make_golden.py).  Runs on the GPU box without
/root/reference."""
import glob
import os

import numpy as np
import pytest

import paper_2601_06849_b200 as etd
from oracle import rel_gap

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CASES = sorted(p for p in glob.glob(os.path.join(GOLD, "*.npz")) if not p.endswith("setup.npz"))
SRC = {1: lambda p: etd.allen_cahn_cubic(), 2: lambda p: etd.poly3(*p[:4]),
       4: lambda p: etd.DeviceSource(etd.SourceKind.AC_MANUFACTURED, tuple(p[:4]), False),
       5: lambda p: etd.singular(p[0]),
       10: lambda p: etd.fhn_cubic(*p[:3]), 11: lambda p: etd.fhn_classic(*p[:2])}


@pytest.mark.parametrize("path", CASES, ids=[os.path.basename(p)[:-4] for p in CASES])
def test_cuda_matches_reference_golden(path):
    z = np.load(path)
    c = {k: z[k] for k in z.files}
    dim, n, steps, fam = int(c["dim"]), int(c["n"]), int(c["steps"]), int(c["family"])
    g = etd.unit_box_grid(dim, n + 1)
    f = SRC[int(c["src_kind"])](list(c["src_params"]))
    if str(c["kind"]) == "scalar":
        plan = etd.make_plan(g, float(c["tau"]), float(c["kappa"]), float(c["q"]), scheme=fam)
        out = etd.advance(plan, etd.StepperState(0, 0.0, c["u0"]), f, nsteps=steps)
        assert rel_gap(c["u"], out.U) <= 1e-11
    else:
        plan = etd.make_system_plan(g, float(c["tau"]), float(c["ku"]), float(c["kv"]), float(c["q"]), scheme=fam)
        out = etd.etd2rkds_step_system(plan, etd.SystemState(0, 0.0, c["u0"], c["v0"]), f, nsteps=steps)
        assert rel_gap(c["u"], out.U) <= 1e-11 and rel_gap(c["v"], out.V) <= 1e-11
    assert out.n == int(c["n_out"]) and out.t == pytest.approx(float(c["t_out"]))
