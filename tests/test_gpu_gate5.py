"""GPU: the reference's release gate 5 (acceptance_main.cpp:172-229) on the device:
for every catalogue problem (allen-cahn-2d/3d, singular-source-2d/3d, fhn-2d) and
both Pade families, the spectral (eigenbasis transforms) and Thomas (tridiagonal
solves) backends stay within 1e-10 of each other in the sup-norm relative gap,
checked after EVERY one of 100 steps at the gate's grid sizes (m = 128 in 2D, 32
in 3D), tau = T/100."""
import numpy as np
import pytest

import paper_2601_06849_b200 as etd
from paper_2601_06849_b200 import harness

pytestmark = pytest.mark.gpu

CASES = [("allen-cahn-2d", 128), ("allen-cahn-3d", 32), ("singular-source-2d", 128), ("singular-source-3d", 32),
         ("fhn-2d", 128)]


def sup_gap(a, b):
    return float(np.max(np.abs(a - b)))


@pytest.mark.parametrize("family", [etd.PadeFamily.P02, etd.PadeFamily.P04], ids=["p02", "p04"])
@pytest.mark.parametrize("problem,m", CASES, ids=[c[0] for c in CASES])
def test_spectral_vs_thomas_every_step(problem, m, family):
    spec = harness.problem_by_name(problem)
    g = etd.unit_box_grid(spec.dim, m)
    N = 100
    tau = spec.T / N
    plans = []
    for backend in (etd.BackendKind.Spectral, etd.BackendKind.Thomas):
        if spec.system:
            p = etd.make_system_plan(g, tau, spec.kappa_u, spec.kappa_v, spec.q, scheme=family, backend=backend,
                                     source=spec.source)
            p.upload(0, spec.initial(g), 0, 0.0)
            p.upload(1, spec.initial_v(g), 0, 0.0)
        else:
            p = etd.make_plan(g, tau, spec.kappa, spec.q, scheme=family, backend=backend, source=spec.source)
            p.upload(0, spec.initial(g), 0, 0.0)
        p.set_source(spec.source)
        plans.append(p)
    worst = 0.0
    ns = 2 if spec.system else 1
    for n in range(N):
        for p in plans:
            p.step(1)
        a = [plans[0].download(s)[0] for s in range(ns)]
        b = [plans[1].download(s)[0] for s in range(ns)]
        num = max(sup_gap(x, y) for x, y in zip(a, b))
        den = max(float(np.max(np.abs(x))) for x in a)
        worst = max(worst, num / den)
    assert plans[0].download(0)[1] == plans[1].download(0)[1] == N
    for p in plans:
        p.close()
    assert worst <= 1e-10, (problem, family, worst)
