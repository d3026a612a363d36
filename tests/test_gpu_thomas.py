"""GPU parity of the Thomas backend (BackendKind::Thomas, reference thomas.cpp)
against the reference's own Thomas path (oracle/_ref) and against the device
spectral backend.

Tolerances: apply_Q_thomas <= 1e-13 relative (same operation order as the
reference, but g++ may contract its complex products into FMAs for C++ at
-march=x86-64-v3, so the last bit is compiler dependent);
full steps normwise <= 1e-11 (BASELINE north_star); spectral vs Thomas
<= 1e-10 over 100 steps (the reference's backend cross-check,
test_stepper.cpp gate 5 / SURVEY.md §4).
"""
import numpy as np
import pytest

import paper_2601_06849_b200 as etd
from oracle import Ref, rel_gap

pytestmark = pytest.mark.gpu

STEP_TOL = 1e-11
needs_ref = pytest.mark.skipif(not Ref.available(), reason="oracle/_ref not built")
TH = etd.BackendKind.Thomas


@needs_ref
@pytest.mark.parametrize("dim,n", [(2, 31), (3, 15), (2, 100), (3, 24), (2, 64), (3, 32), (2, 8), (3, 4)])
@pytest.mark.parametrize("family", [0, 1])
def test_apply_q_thomas_vs_reference(dim, n, family):
    tau, kappa, q = 0.02, 0.7, 1.0
    g = etd.unit_box_grid(dim, n + 1)
    plan = etd.make_plan(g, tau, kappa, q, scheme=family, backend=TH, source=etd.allen_cahn_cubic())
    x = np.random.default_rng(2).uniform(-0.5, 0.5, n ** dim)
    for axis in range(dim):
        for ell in (1, 2, 3):
            got = plan.debug_transform(x, axis, ell=ell, apply_q=True)
            want = Ref.apply_q_thomas(dim, n, tau, kappa, q, family, ell, axis, x)
            scale = np.max(np.abs(want))
            assert np.max(np.abs(got - want)) <= 1e-13 * scale, (axis, ell)


@needs_ref
@pytest.mark.parametrize("dim,n,steps", [(2, 63, 10), (3, 31, 5), (2, 9, 3), (3, 20, 4)])
@pytest.mark.parametrize("family", [0, 1])
def test_thomas_scalar_steps_vs_reference(dim, n, steps, family):
    tau, kappa, q = 0.01, 1.0, 1.0
    g = etd.unit_box_grid(dim, n + 1)
    u0 = np.random.default_rng(3).uniform(-1, 1, n ** dim)
    plan = etd.make_plan(g, tau, kappa, q, scheme=family, backend=TH)
    assert plan.backend == etd.BackendKind.CudaThomas
    got = etd.advance(plan, etd.StepperState(0, 0.0, u0), etd.allen_cahn_cubic(), nsteps=steps)
    want, nn, tt = Ref.scalar_run(dim, n, tau, kappa, q, u0, steps, src_kind=1, family=family, backend=1)[:3]
    assert got.n == nn == steps and got.t == pytest.approx(tt)
    assert rel_gap(want, got.U) <= STEP_TOL


@needs_ref
@pytest.mark.parametrize("dim,n,steps", [(2, 63, 6), (3, 31, 4), (3, 17, 3)])
@pytest.mark.parametrize("family", [0, 1])
def test_thomas_system_steps_vs_reference(dim, n, steps, family):
    """2D: the reference's make_system_plan(..., Thomas); 3D: the same step with
    the z->y filter (oracle composition of reference calls)."""
    tau, ku, kv = 0.05, 1e-3, 5e-4
    rng = np.random.default_rng(4)
    u0, v0 = rng.uniform(-1, 1, n ** dim), rng.uniform(-1, 1, n ** dim)
    g = etd.unit_box_grid(dim, n + 1)
    plan = etd.make_system_plan(g, tau, ku, kv, 0.0, scheme=family, backend=TH)
    f = etd.fhn_cubic(0.1, 0.01, 0.5)
    got = etd.etd2rkds_step_system(plan, etd.SystemState(0, 0.0, u0, v0), f, nsteps=steps)
    wu, wv, nn, tt = Ref.system_run(dim, n, tau, ku, kv, 0.0, u0, v0, steps, src_kind=10,
                                    src_params=(0.1, 0.01, 0.5), family=family, backend=1)[:4]
    assert got.n == nn
    assert rel_gap(wu, got.U) <= STEP_TOL and rel_gap(wv, got.V) <= STEP_TOL


@needs_ref
@pytest.mark.parametrize("dim,n,steps", [(2, 47, 6), (3, 21, 4)])
def test_thomas_manufactured_and_singular_vs_reference(dim, n, steps):
    g = etd.unit_box_grid(dim, n + 1)
    src = etd.allen_cahn_manufactured(dim, 1.0, 1.0)
    u0 = np.random.default_rng(21).uniform(0.0, 0.8, n ** dim)
    plan = etd.make_plan(g, 0.01, 1.0, 0.0, backend=TH)
    got = etd.advance(plan, etd.StepperState(3, 0.03, u0), src, nsteps=steps)
    want = Ref.scalar_run(dim, n, 0.01, 1.0, 0.0, u0, steps, src_kind=4, src_params=src.params8(), backend=1,
                          n0=3, t0=0.03)[0]
    assert rel_gap(want, got.U) <= STEP_TOL
    u1 = 0.5 * u0
    got = etd.advance(plan, etd.StepperState(0, 0.0, u1), etd.singular(0.1), nsteps=steps)
    want = Ref.scalar_run(dim, n, 0.01, 1.0, 0.0, u1, steps, src_kind=5, src_params=(0.1,), backend=1)[0]
    assert rel_gap(want, got.U) <= STEP_TOL


@pytest.mark.parametrize("dim,m,family", [(2, 128, 0), (2, 96, 1), (3, 32, 0)])
def test_spectral_vs_thomas_cross_check(dim, m, family):
    """Both device backends agree within 1e-10 over 100 steps (the reference's
    spectral-vs-thomas gate)."""
    g = etd.unit_box_grid(dim, m)
    n = m - 1
    u0 = np.random.default_rng(8).uniform(-1, 1, n ** dim)
    st = etd.StepperState(0, 0.0, u0)
    a = etd.advance(etd.make_plan(g, 0.005, 1.0, 1.0, scheme=family), st, etd.allen_cahn_cubic(), nsteps=100)
    b = etd.advance(etd.make_plan(g, 0.005, 1.0, 1.0, scheme=family, backend=TH), st, etd.allen_cahn_cubic(),
                    nsteps=100)
    assert a.n == b.n == 100
    assert rel_gap(a.U, b.U) <= 1e-10


@pytest.mark.parametrize("shape,family", [((47, 31, 63), 0), ((40, 130, 9), 1), ((70, 37), 0)])
def test_thomas_ragged_grids_vs_spectral(shape, family):
    """Non-cubic grids: pencil counts that leave partial 128- / 64-pencil tiles, axis
    extents that are not multiples of the 8-point chunks (guarded edge chunks next to
    the 16- / 32-byte interior accesses), two species and one.  The two device
    backends agree within the reference's cross-check tolerance."""
    dim = len(shape)
    g = etd.build_grid(dim, [(0.0, 1.0)] * dim, [s + 1 for s in shape])
    N = int(np.prod(shape))
    rng = np.random.default_rng(31)
    u0, v0 = rng.uniform(-1, 1, N), rng.uniform(-1, 1, N)
    f = etd.fhn_cubic(0.1, 0.01, 0.5)
    st2 = etd.SystemState(0, 0.0, u0, v0)
    a = etd.etd2rkds_step_system(etd.make_system_plan(g, 0.05, 1e-3, 5e-4, 0.0, scheme=family), st2, f, nsteps=20)
    b = etd.etd2rkds_step_system(etd.make_system_plan(g, 0.05, 1e-3, 5e-4, 0.0, scheme=family, backend=TH), st2, f,
                                 nsteps=20)
    assert a.n == b.n == 20
    assert rel_gap(a.U, b.U) <= 1e-10 and rel_gap(a.V, b.V) <= 1e-10
    st1 = etd.StepperState(0, 0.0, u0)
    c = etd.advance(etd.make_plan(g, 0.005, 1.0, 1.0, scheme=family), st1, etd.allen_cahn_cubic(), nsteps=20)
    d = etd.advance(etd.make_plan(g, 0.005, 1.0, 1.0, scheme=family, backend=TH), st1, etd.allen_cahn_cubic(),
                    nsteps=20)
    assert rel_gap(c.U, d.U) <= 1e-10


def test_thomas_abort_semantics():
    """Non-finite source -> StepperAbort(input t, n) with the input state kept;
    domain violation -> step -1 (same contract as the spectral backend)."""
    g = etd.unit_box_grid(2, 8)
    plan = etd.make_plan(g, 0.01, 1.0, 1.0, backend=TH)
    u0 = np.random.default_rng(7).uniform(-0.5, 0.5, 49)
    with pytest.raises(etd.StepperAbort) as ei:
        etd.advance(plan, etd.StepperState(4, 0.25, u0), etd.DeviceSource(etd.SourceKind.NAN_PROBE))
    assert ei.value.t == pytest.approx(0.25) and ei.value.step == 4
    u, n, t = plan.download(0)
    assert n == 4 and np.array_equal(u, u0)
    bad = 0.5 * np.abs(u0)
    bad[7] = 1.0
    with pytest.raises(etd.StepperAbort) as ei:
        etd.advance(plan, etd.StepperState(2, 0.02, bad), etd.singular(0.1), nsteps=3)
    assert ei.value.step == -1
    # a diverging run stops at the failing step with the last good state
    plan2 = etd.make_plan(etd.unit_box_grid(2, 16), 0.5, 1e-3, 0.0, backend=TH)
    with pytest.raises(etd.StepperAbort) as ei:
        etd.advance(plan2, etd.StepperState(0, 0.0, np.full(225, 3.0)), etd.poly3(0.0, 0.0, 0.0, 1e6), nsteps=50)
    u, n, t = plan2.download(0)
    assert n == ei.value.step and np.all(np.isfinite(u))


def test_thomas_plan_rejections():
    g3 = etd.unit_box_grid(3, 16)
    with pytest.raises(etd.ConfigError):
        etd.StepperPlan(g3, 0.01, 1.0, 0.0, world_size=2, rank=0, backend=TH)
    with pytest.raises(etd.ConfigError):
        etd.make_plan(g3, 0.01, 1.0, 0.0, backend=etd.BackendKind.NonSplitBanded)
    plan = etd.make_plan(etd.unit_box_grid(2, 16), 0.01, 1.0, 0.0, backend=TH)
    with pytest.raises(etd.ConfigError):
        plan.debug_transform(np.zeros(225), 0, back=True)  # only apply_Q on Thomas plans


def test_thomas_profiling_and_graph_paths_agree():
    g = etd.unit_box_grid(3, 24)
    u0 = np.random.default_rng(9).uniform(-1, 1, 23 ** 3)
    out = []
    for prof in (False, True):
        plan = etd.make_plan(g, 0.01, 1.0, 1.0, backend=TH)
        plan.set_profiling(prof)
        plan.upload(0, u0)
        plan.step(5)
        out.append(plan.download(0)[0])
        if prof:
            names = [s["name"] for s in plan.stage_stats()]
            assert names == ["source", "thomas_z", "thomas_y", "thomas_x_what", "thomas_x_upd"]
    assert np.array_equal(out[0], out[1])
