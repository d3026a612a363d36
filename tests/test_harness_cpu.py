"""CPU: the study-harness file formats against files written by the reference
harness itself (tests/golden/harness/, made by tests/golden/make_golden_harness.py):
the ETRJ reference-trajectory cache with its JSON fingerprint
(harness.cpp:49-115, 135-149) and the convergence CSV (harness.cpp:364-421)."""
import os
import shutil

import numpy as np
import pytest

import paper_2601_06849_b200 as etd
from paper_2601_06849_b200 import harness

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "harness")
CASES = [("singular-source-2d", 16, 0, 16), ("fhn-2d", 16, 0, 16), ("singular-source-3d", 8, 1, 10)]


def traj_path(problem, m, fam):
    spec = harness.problem_by_name(problem)
    return spec, os.path.join(GOLD, os.path.basename(harness.reference_path("", spec, m, fam)))


@pytest.mark.parametrize("problem,m,fam,coarse", CASES)
def test_etrj_reference_file_roundtrip(problem, m, fam, coarse, tmp_path):
    spec, path = traj_path(problem, m, fam)
    g = etd.unit_box_grid(spec.dim, m)
    fp = harness.param_fingerprint(spec, harness.ProblemParams(), coarse, etd.BackendKind.Spectral)
    ncomp = 2 if spec.system else 1
    got = harness.read_traj_file(path, fp, spec.dim, g.interior_shape(), ncomp)
    assert got is not None
    times, comps = got
    assert len(times) == coarse + 1 and times[0] == 0.0 and times[-1] == pytest.approx(spec.T)
    assert all(c.shape == (g.total_interior(),) for comp in comps for c in comp)
    if not spec.system:
        assert np.array_equal(comps[0][0], spec.initial(g))  # the reference's initial_u, bitwise
    # our writer reproduces the reference's bytes (fingerprint text included)
    out = str(tmp_path / "x.traj")
    harness.write_traj_file(out, fp, times, comps, spec.dim, g.interior_shape())
    assert open(out, "rb").read() == open(path, "rb").read()
    # a stale fingerprint, a wrong shape or a truncated file invalidate the cache
    bad = dict(fp, rho=0.2)
    assert harness.read_traj_file(path, bad, spec.dim, g.interior_shape(), ncomp) is None
    assert harness.read_traj_file(path, fp, spec.dim, (1, 2, 3), ncomp) is None
    short = str(tmp_path / "short.traj")
    open(short, "wb").write(open(path, "rb").read()[:-8])
    assert harness.read_traj_file(short, fp, spec.dim, g.interior_shape(), ncomp) is None
    assert harness.read_traj_file(str(tmp_path / "missing.traj"), fp, spec.dim, g.interior_shape(), ncomp) is None


@pytest.mark.parametrize("problem,m,fam,coarse", CASES)
def test_convergence_csv_reference_roundtrip(problem, m, fam, coarse, tmp_path):
    name = f"convergence_{problem}_{'p04' if fam else 'p02'}_spectral_m{m}.csv"
    src = os.path.join(GOLD, name)
    rep = harness.parse_convergence_csv(src)
    assert rep.problem == problem and rep.m == m and rep.backend == "spectral" and len(rep.rows) == 2
    assert rep.rows[0].eoc is None and rep.rows[1].eoc == pytest.approx(np.log2(rep.rows[0].E / rep.rows[1].E))
    out = str(tmp_path / name)
    harness.write_convergence_csv(rep, out)
    assert open(out).read() == open(src).read()


def test_problem_catalogue_and_guards():
    assert harness.problem_names() == ["allen-cahn-2d", "allen-cahn-3d", "singular-source-2d",
                                       "singular-source-3d", "fhn-2d"]
    for n in harness.problem_names():
        s = harness.problem_by_name(n)
        assert s.name == n and (s.has_exact or s.reference_N > 0)
    with pytest.raises(etd.ConfigError):
        harness.problem_by_name("heat-2d")
    with pytest.raises(etd.ConfigError):
        harness.integrate_scalar(harness.allen_cahn(2), None, 10, 3)
    with pytest.raises(etd.ConfigError):
        harness.compute_error_E(harness.Trajectory([0.0], [np.zeros(4)]), harness.Trajectory([0.0, 1.0], []))
