"""GPU: the device study harness against files written by the reference
harness (tests/golden/harness/): fine-N reference trajectories (ETRJ cache,
harness.cpp:252-283) and convergence tables E(N) (harness.cpp:305-362) for the
catalogue problems without a closed form (singular source 2D/3D, FitzHugh-Nagumo 2D)."""
import os
import shutil

import numpy as np
import pytest

import paper_2601_06849_b200 as etd
from paper_2601_06849_b200 import harness
from oracle import rel_gap

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "harness")
CASES = [("singular-source-2d", 16, 0, 16, (16, 32)), ("fhn-2d", 16, 0, 16, (16, 32)),
         ("singular-source-3d", 8, 1, 10, (10, 20))]


def golden_traj(spec, m, fam, coarse):
    g = etd.unit_box_grid(spec.dim, m)
    fp = harness.param_fingerprint(spec, harness.ProblemParams(), coarse, etd.BackendKind.Spectral)
    path = os.path.join(GOLD, os.path.basename(harness.reference_path("", spec, m, fam)))
    return harness.read_traj_file(path, fp, spec.dim, g.interior_shape(), 2 if spec.system else 1), path


@pytest.mark.parametrize("backend", [etd.BackendKind.Spectral, etd.BackendKind.Thomas])
@pytest.mark.parametrize("problem,m,fam,coarse,Ns", CASES)
def test_reference_trajectory_vs_reference_harness(problem, m, fam, coarse, Ns, backend):
    spec = harness.problem_by_name(problem)
    (times, comps), _ = golden_traj(spec, m, fam, coarse)
    ref = harness.truth_trajectory(spec, m, coarse, fam, backend)
    mine = [ref.u, ref.v] if spec.system else [ref.fields]
    assert np.allclose(ref.times, times, rtol=0, atol=1e-12)
    for a, b in zip(mine, comps):
        for x, y in zip(a, b):
            assert rel_gap(y, x) <= 1e-11


@pytest.mark.parametrize("problem,m,fam,coarse,Ns", CASES)
def test_convergence_table_vs_reference_harness(problem, m, fam, coarse, Ns, tmp_path):
    spec = harness.problem_by_name(problem)
    out = str(tmp_path)
    rows = harness.run_convergence(spec, m, list(Ns), scheme=fam, coarse=coarse, out=out)
    gold = harness.parse_convergence_csv(
        os.path.join(GOLD, f"convergence_{problem}_{'p04' if fam else 'p02'}_spectral_m{m}.csv"))
    for r, g in zip(rows, gold.rows):
        assert r.N == g.N and abs(r.E - g.E) <= 1e-9 * g.E
    mine = harness.parse_convergence_csv(
        os.path.join(out, f"convergence_{problem}_{'p04' if fam else 'p02'}_spectral_m{m}.csv"))
    assert [r.N for r in mine.rows] == list(Ns)
    # the cache we wrote is a valid reference cache file
    (times, comps), gpath = golden_traj(spec, m, fam, coarse)
    fp = harness.param_fingerprint(spec, harness.ProblemParams(), coarse, etd.BackendKind.Spectral)
    got = harness.read_traj_file(harness.reference_path(out, spec, m, fam), fp, spec.dim,
                                 etd.unit_box_grid(spec.dim, m).interior_shape(), len(comps))
    assert got is not None and rel_gap(comps[0][-1], got[1][0][-1]) <= 1e-11


def test_cached_reference_trajectory_is_used(tmp_path):
    """A cache file with a matching fingerprint replaces the fine-N run
    (harness.cpp:257-260): a perturbed cached truth moves E."""
    spec = harness.problem_by_name("singular-source-2d")
    (times, comps), _ = golden_traj(spec, 16, 0, 16)
    fp = harness.param_fingerprint(spec, harness.ProblemParams(), 16, etd.BackendKind.Spectral)
    out = str(tmp_path)
    bumped = [[c + 1e-3 for c in comps[0]]]
    harness.write_traj_file(harness.reference_path(out, spec, 16, 0), fp, times, bumped, 2, (15, 15, 1))
    E_cached = harness.run_convergence(spec, 16, [16], coarse=16, out=out)[0].E
    E_fresh = harness.run_convergence(spec, 16, [16], coarse=16)[0].E
    assert abs(E_cached - E_fresh) > 5e-4
