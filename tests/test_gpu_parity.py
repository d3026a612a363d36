"""GPU parity: the CUDA path (through the C-ABI) against the reference itself
(oracle/_ref, the unmodified etdrd core) and the C restatement (oracle/).

Tolerances follow the reference's own tests: contraction vs naive <= 1e-13
(test_tensor.cpp:45-71), apply_Q <= 1e-12 (test_tensor.cpp:105-125), steps
normwise max|a-b|/max|a| <= 1e-11 (BASELINE north_star; rel_gap of
test_stepper.cpp:50-57).
"""
import numpy as np
import pytest

import paper_2601_06849_b200 as etd
from paper_2601_06849_b200 import configs
from oracle import Oracle, Ref, rel_gap

pytestmark = pytest.mark.gpu

STEP_TOL = 1e-11


def ref_or_oracle():
    return Ref if Ref.available() else Oracle


def sine_mode(g):
    nx, ny, nz = g.interior_shape()
    x = np.sin(np.pi * np.array([g.coord(0, i) for i in range(nx)]))
    y = np.sin(np.pi * np.array([g.coord(1, j) for j in range(ny)]))
    z = np.sin(np.pi * np.array([g.coord(2, k) for k in range(nz)])) if g.dim == 3 else np.ones(1)
    return (z[:, None, None] * y[None, :, None] * x[None, None, :]).ravel()


# ----------------------------------------------------------------- transforms
@pytest.mark.parametrize("shape", [(45, 33, 1), (21, 17, 13), (127, 127, 1), (64, 48, 40), (7, 9, 5)])
def test_transform_vs_reference_contract(shape):
    nx, ny, nz = shape
    dim = 3 if nz > 1 else 2
    g = etd.build_grid(dim, [(0.0, 1.0)] * dim, [s + 1 for s in shape[:dim]])
    plan = etd.make_plan(g, 0.01, 1.0, 1.0, source=etd.allen_cahn_cubic())
    rng = np.random.default_rng(1)
    x = rng.uniform(-1, 1, nx * ny * nz)
    for axis in range(dim):
        n = shape[axis]
        P, _ = Oracle.spectral_factor(n, 2.0, -1.0)   # P is independent of diag/off
        for back in (False, True):
            got = plan.debug_transform(x, axis, back=back)
            want = Ref.contract_axis(shape, P, n, x, axis, transpose=not back) if Ref.available() \
                else Oracle.contract(shape, P, x, axis, transpose=not back)
            assert np.max(np.abs(got - want)) <= 1e-13, (shape, axis, back)


@pytest.mark.parametrize("dim,n", [(2, 31), (3, 15), (2, 100)])
@pytest.mark.parametrize("family", [0, 1])
def test_apply_q_vs_reference(dim, n, family):
    tau, kappa, q = 0.02, 0.7, 1.0
    g = etd.unit_box_grid(dim, n + 1)
    plan = etd.make_plan(g, tau, kappa, q, scheme=family, source=etd.allen_cahn_cubic())
    x = np.random.default_rng(2).uniform(-0.5, 0.5, n ** dim)
    for axis in range(dim):
        for ell in (1, 2, 3):
            got = plan.debug_transform(x, axis, ell=ell, apply_q=True)
            want = ref_or_oracle().apply_q(dim, n, tau, kappa, q, family, ell, axis, x)
            assert np.max(np.abs(got - want)) <= 1e-12, (axis, ell)


# ----------------------------------------------------------------- full steps
@pytest.mark.parametrize("dim,n,steps", [(2, 63, 10), (3, 31, 5), (2, 9, 3), (3, 20, 4)])
@pytest.mark.parametrize("family", [0, 1])
def test_scalar_steps_vs_reference(dim, n, steps, family):
    tau, kappa, q = 0.01, 1.0, 1.0
    g = etd.unit_box_grid(dim, n + 1)
    u0 = np.random.default_rng(3).uniform(-1, 1, n ** dim)
    plan = etd.make_plan(g, tau, kappa, q, scheme=family)
    got = etd.advance(plan, etd.StepperState(0, 0.0, u0), etd.allen_cahn_cubic(), nsteps=steps)
    want, nn, tt = ref_or_oracle().scalar_run(dim, n, tau, kappa, q, u0, steps, src_kind=1, family=family)[:3]
    assert got.n == nn == steps and got.t == pytest.approx(tt)
    assert rel_gap(want, got.U) <= STEP_TOL


@pytest.mark.parametrize("dim,n,steps", [(2, 63, 6), (3, 31, 4), (3, 17, 3)])
@pytest.mark.parametrize("src", ["fhn_cubic", "fhn_classic"])
@pytest.mark.parametrize("q", [0.0, 0.8])
def test_system_steps_vs_reference(dim, n, steps, src, q):
    """Two species against the reference: 2D through its make_system_plan, 3D the
    composed step.  q != 0 checks that kappa_c scales the unit-kappa eigenvalue
    with its q/dim term (system_stepper.cpp:52-61)."""
    tau, ku, kv = 0.05, 2e-2 if q else 1e-3, 5e-4
    rng = np.random.default_rng(4)
    u0, v0 = rng.uniform(-1, 1, n ** dim), rng.uniform(-1, 1, n ** dim)
    if src == "fhn_cubic":
        f, kind, params = etd.fhn_cubic(0.1, 0.01, 0.5), 10, (0.1, 0.01, 0.5)
    else:
        f, kind, params = etd.fhn_classic(1.0, 1.0), 11, (1.0, 1.0)
    g = etd.unit_box_grid(dim, n + 1)
    plan = etd.make_system_plan(g, tau, ku, kv, q)
    got = etd.etd2rkds_step_system(plan, etd.SystemState(0, 0.0, u0, v0), f, nsteps=steps)
    wu, wv, nn, tt = ref_or_oracle().system_run(dim, n, tau, ku, kv, q, u0, v0, steps, src_kind=kind,
                                                 src_params=params)[:4]
    assert got.n == nn
    assert rel_gap(wu, got.U) <= STEP_TOL and rel_gap(wv, got.V) <= STEP_TOL


@pytest.mark.parametrize("cfg_id,n,steps", [(0, 127, 100), (1, 255, 10), (2, 63, 10), (3, 47, 5), (4, 31, 5)])
def test_config_shapes_vs_reference(cfg_id, n, steps):
    """BASELINE configs with their own kappa/q/tau/source and seeded inputs, at
    sizes the CPU reference finishes in seconds (config 0 at full size)."""
    cfg = configs.CONFIGS[cfg_id]
    ics = configs.initial_state(cfg, n)
    plan = configs.make_plan(cfg, n)
    R = ref_or_oracle()
    if cfg.nspecies == 1:
        got = etd.advance(plan, etd.StepperState(0, 0.0, ics[0]), cfg.source, nsteps=steps)
        want = R.scalar_run(cfg.dim, n, cfg.tau, cfg.kappa[0], cfg.q, ics[0], steps, src_kind=1)[0]
        assert rel_gap(want, got.U) <= STEP_TOL
    else:
        got = etd.etd2rkds_step_system(plan, etd.SystemState(0, 0.0, ics[0], ics[1]), cfg.source, nsteps=steps)
        wu, wv = R.system_run(cfg.dim, n, cfg.tau, cfg.kappa[0], cfg.kappa[1], cfg.q, ics[0], ics[1], steps,
                              src_kind=10, src_params=(0.1, 0.01, 0.5))[:2]
        assert rel_gap(wu, got.U) <= STEP_TOL and rel_gap(wv, got.V) <= STEP_TOL


@pytest.mark.parametrize("cfg_id,n,steps", [(3, 127, 3), (2, 127, 4), (1, 767, 6)])
def test_default_level2_schedule_vs_reference(cfg_id, n, steps):
    """BASELINE physics at sizes where the default plan picks the second-level split
    by itself (>= 2^18 points, n = 32m - 1): the shipped schedule, not a forced
    one, against the reference CPU implementation."""
    cfg = configs.CONFIGS[cfg_id]
    plan = configs.make_plan(cfg, n)
    assert plan.fold_level()[:cfg.dim] == (2,) * cfg.dim
    ics = configs.initial_state(cfg, n)
    R = ref_or_oracle()
    if cfg.nspecies == 1:
        got = etd.advance(plan, etd.StepperState(0, 0.0, ics[0]), cfg.source, nsteps=steps)
        want = R.scalar_run(cfg.dim, n, cfg.tau, cfg.kappa[0], cfg.q, ics[0], steps, src_kind=1)[0]
        assert rel_gap(want, got.U) <= STEP_TOL
    else:
        got = etd.etd2rkds_step_system(plan, etd.SystemState(0, 0.0, ics[0], ics[1]), cfg.source, nsteps=steps)
        wu, wv = R.system_run(cfg.dim, n, cfg.tau, cfg.kappa[0], cfg.kappa[1], cfg.q, ics[0], ics[1], steps,
                              src_kind=10, src_params=(0.1, 0.01, 0.5))[:2]
        assert rel_gap(wu, got.U) <= STEP_TOL and rel_gap(wv, got.V) <= STEP_TOL


# ----------------------------------------------------------------- semantics
def test_zero_source_sine_mode_scalar_weights():
    """test_stepper.cpp:109-126"""
    g = etd.unit_box_grid(2, 10)
    tau, kappa, q = 0.02, 1.3, 0.7
    u0 = sine_mode(g)
    for fam in (0, 1):
        plan = etd.make_plan(g, tau, kappa, q, scheme=fam)
        out = etd.advance(plan, etd.StepperState(0, 0.0, u0), etd.DeviceSource(etd.SourceKind.ZERO))
        sch = etd.setup_scheme(fam)
        lam = []
        for a in range(2):
            _, l = etd.setup_axis(9, kappa, q, 2)
            lam.append(l[0])
        w = 1.0
        for lv in lam:
            x = tau * lv
            w *= 2.0 * sum(np.real(complex(t[2], t[3]) / (x - complex(t[0], t[1]))) for t in sch[0])
        assert np.max(np.abs(out.U - w * u0)) <= 1e-12


def test_nonfinite_source_aborts_with_input_state():
    """test_stepper.cpp:304-321: StepperAbort carries the INPUT state's t and n."""
    g = etd.unit_box_grid(2, 8)
    plan = etd.make_plan(g, 0.01, 1.0, 1.0)
    u0 = np.random.default_rng(7).uniform(-0.5, 0.5, 49)
    with pytest.raises(etd.StepperAbort) as ei:
        etd.advance(plan, etd.StepperState(4, 0.25, u0), etd.DeviceSource(etd.SourceKind.NAN_PROBE))
    assert ei.value.t == pytest.approx(0.25) and ei.value.step == 4
    # the device state is the input of the failing step (nothing committed)
    u, n, t = plan.download(0)
    assert n == 4 and np.array_equal(u, u0)


def test_abort_mid_run_keeps_last_good_state():
    """A run that blows up at step k reports step k and keeps the state after k steps."""
    g = etd.unit_box_grid(2, 16)
    plan = etd.make_plan(g, 0.5, 1e-3, 0.0)
    u0 = np.full(15 * 15, 3.0)  # u - u^3 with a huge tau diverges within a few steps
    st = etd.StepperState(0, 0.0, u0)
    with pytest.raises(etd.StepperAbort) as ei:
        etd.advance(plan, st, etd.poly3(0.0, 0.0, 0.0, 1e6), nsteps=50)
    k = ei.value.step
    assert 0 <= k < 50
    u, n, t = plan.download(0)
    assert n == k and np.all(np.isfinite(u))
    # replaying k steps from the start reproduces that state bitwise
    plan2 = etd.make_plan(g, 0.5, 1e-3, 0.0)
    if k > 0:
        again = etd.advance(plan2, st, etd.poly3(0.0, 0.0, 0.0, 1e6), nsteps=k)
        assert np.array_equal(again.U, u)


def test_bitwise_reproducible_and_batched_equals_single():
    """test_stepper.cpp:323-332 plus advance(n) == n x advance(1)."""
    g = etd.unit_box_grid(3, 24)
    plan = etd.make_plan(g, 0.01, 0.5, 1.0, scheme=1)
    u0 = np.random.default_rng(8).uniform(-1, 1, 23 ** 3)
    st = etd.StepperState(0, 0.0, u0)
    a = etd.advance(plan, st, etd.allen_cahn_cubic())
    b = etd.advance(plan, st, etd.allen_cahn_cubic())
    assert np.array_equal(a.U, b.U)
    five = etd.advance(plan, st, etd.allen_cahn_cubic(), nsteps=5)
    s = st
    for _ in range(5):
        s = etd.advance(plan, s, etd.allen_cahn_cubic())
    assert np.array_equal(five.U, s.U) and five.n == s.n == 5


def test_mirrored_system_keeps_v_equal_u():
    """test_stepper.cpp:430-446"""
    for dim, n in ((2, 9), (3, 11)):
        g = etd.unit_box_grid(dim, n + 1)
        u0 = np.random.default_rng(31).uniform(-0.5, 0.5, n ** dim)
        plan = etd.make_system_plan(g, 0.02, 0.5, 0.5, 0.0, scheme=1)
        st = etd.etd2rkds_step_system(plan, etd.SystemState(0, 0.0, u0, u0),
                                      etd.DeviceSource(etd.SourceKind.MIRROR_AC), nsteps=10)
        assert np.max(np.abs(st.U - st.V)) <= 1e-12


def test_decoupled_system_equals_two_scalar_runs():
    """test_stepper.cpp:448-488 (autonomous v source), in 2D and 3D."""
    for dim, n in ((2, 9), (3, 9)):
        g = etd.unit_box_grid(dim, n + 1)
        tau, ku, kv = 0.01, 0.05, 2.0
        rng = np.random.default_rng(11)
        u0, v0 = rng.uniform(-0.5, 0.5, n ** dim), rng.uniform(-0.5, 0.5, n ** dim)
        sp = etd.make_system_plan(g, tau, ku, kv, 0.0)
        st = etd.etd2rkds_step_system(sp, etd.SystemState(0, 0.0, u0, v0),
                                      etd.DeviceSource(etd.SourceKind.DECOUPLED, (-0.3, 0.1)), nsteps=8)
        pu = etd.make_plan(g, tau, ku, 0.0)
        pv = etd.make_plan(g, tau, kv, 0.0)
        au = etd.advance(pu, etd.StepperState(0, 0.0, u0), etd.allen_cahn_cubic(), nsteps=8)
        av = etd.advance(pv, etd.StepperState(0, 0.0, v0), etd.poly3(0.1, -0.3), nsteps=8)
        assert np.max(np.abs(st.U - au.U)) <= 1e-12
        assert np.max(np.abs(st.V - av.U)) <= 1e-12


def test_shape_mismatch_and_host_source_rejected():
    g = etd.unit_box_grid(2, 8)
    plan = etd.make_plan(g, 0.01, 1.0, 1.0)
    with pytest.raises(etd.ConfigError):
        etd.advance(plan, etd.StepperState(0, 0.0, np.zeros(64)), etd.allen_cahn_cubic())
    with pytest.raises(etd.ConfigError):
        etd.advance(plan, etd.StepperState(0, 0.0, np.zeros(49)), lambda t, u, g: u)
    with pytest.raises(etd.ConfigError):
        etd.make_plan(g, 0.0, 1.0, 1.0)


def test_pipelined_advance_equals_device_resident_steps():
    """etd_advance (H2D/D2H pipelined against the first/last kernels, chunked
    launches, deferred commit) is bitwise equal to upload + etd_step + download."""
    grid = etd.build_grid(3, [(0, 1)] * 3, [30, 26, 40])
    nx, ny, nz = grid.interior_shape()
    rng = np.random.default_rng(12)
    u0, v0 = rng.uniform(-1, 1, nx * ny * nz), rng.uniform(-0.5, 0.5, nx * ny * nz)
    f = etd.fhn_cubic()
    for steps in (1, 3):
        plan = etd.make_system_plan(grid, 0.05, 1e-3, 5e-4, 0.0)
        a = etd.etd2rkds_step_system(plan, etd.SystemState(2, 0.1, u0, v0), f, nsteps=steps)
        plan2 = etd.make_system_plan(grid, 0.05, 1e-3, 5e-4, 0.0, source=f)
        plan2.upload(0, u0, 2, 0.1)
        plan2.upload(1, v0, 2, 0.1)
        plan2.step(steps)
        bu, n, t = plan2.download(0)
        bv, _, _ = plan2.download(1)
        assert np.array_equal(a.U, bu) and np.array_equal(a.V, bv)
        assert a.n == n == 2 + steps and a.t == pytest.approx(t)


@pytest.mark.parametrize("pin_in,pin_out", [(True, True), (False, True), (True, False), (False, False)])
def test_pipelined_advance_pinned_and_pageable_buffers(pin_in, pin_out, monkeypatch):
    """The pipelined advance DMAs pinned host buffers directly and stages pageable
    ones (plain numpy, the reference Field's std::vector) through the plan's pinned
    mirror with host copy threads: every mix of the two is bitwise equal to the
    device-resident steps, and the caller's input is left untouched."""
    import torch
    monkeypatch.setenv("ETD_COPY_THREADS", "3")
    grid = etd.build_grid(3, [(0, 1)] * 3, [40, 34, 30])
    nx, ny, nz = grid.interior_shape()
    rng = np.random.default_rng(5)
    u0, v0 = rng.uniform(-1, 1, nx * ny * nz), rng.uniform(-0.5, 0.5, nx * ny * nz)
    f = etd.fhn_cubic()
    ref = etd.make_system_plan(grid, 0.05, 1e-3, 5e-4, 0.0, source=f)
    ref.upload(0, u0, 0, 0.0)
    ref.upload(1, v0, 0, 0.0)
    ref.step(2)
    wu, wv = ref.download(0)[0], ref.download(1)[0]

    def buf(a, pinned):
        t = torch.from_numpy(a.copy())
        return t.pin_memory() if pinned else t

    hin = [buf(u0, pin_in), buf(v0, pin_in)]
    hout = [buf(np.zeros_like(u0), pin_out), buf(np.zeros_like(v0), pin_out)]
    plan = etd.make_system_plan(grid, 0.05, 1e-3, 5e-4, 0.0, source=f)
    n, t = plan.advance_ptr(hin[0].data_ptr(), hin[1].data_ptr(), hout[0].data_ptr(), hout[1].data_ptr(), 0, 0.0, 2)
    assert n == 2
    assert np.array_equal(hout[0].numpy(), wu) and np.array_equal(hout[1].numpy(), wv)
    assert np.array_equal(hin[0].numpy(), u0) and np.array_equal(hin[1].numpy(), v0)


def test_pipelined_advance_abort_3d():
    g = etd.unit_box_grid(3, 14)
    plan = etd.make_plan(g, 0.01, 1.0, 1.0)
    u0 = np.random.default_rng(3).uniform(-0.5, 0.5, 13 ** 3)
    with pytest.raises(etd.StepperAbort) as ei:
        etd.advance(plan, etd.StepperState(9, 0.09, u0), etd.DeviceSource(etd.SourceKind.NAN_PROBE), nsteps=3)
    assert ei.value.step == 9 and ei.value.t == pytest.approx(0.09)
    u, n, t = plan.download(0)
    assert n == 9 and np.array_equal(u, u0)


@pytest.mark.parametrize("dim,n,steps", [(2, 47, 6), (3, 21, 4)])
def test_manufactured_allen_cahn_vs_reference(dim, n, steps):
    """Catalogue Allen-Cahn source (non-autonomous, position dependent) against
    the reference's own allen_cahn().source (problems.cpp:68-106)."""
    g = etd.unit_box_grid(dim, n + 1)
    src = etd.allen_cahn_manufactured(dim, 1.0, 1.0)
    u0 = np.random.default_rng(21).uniform(0.0, 0.8, n ** dim)
    for fam in (0, 1):
        plan = etd.make_plan(g, 0.01, 1.0, 0.0, scheme=fam)
        got = etd.advance(plan, etd.StepperState(3, 0.03, u0), src, nsteps=steps)
        want = ref_or_oracle().scalar_run(dim, n, 0.01, 1.0, 0.0, u0, steps, src_kind=4,
                                          src_params=src.params8(), family=fam, n0=3, t0=0.03)[0]
        assert rel_gap(want, got.U) <= STEP_TOL


def test_singular_source_vs_reference_and_domain_abort():
    """rho u/(1-u) (problems.cpp:108-136) and its domain guard: u >= 1 aborts
    with StepperAbort(t, step = -1) and the input state kept."""
    n = 31
    for dim in (2, 3):
        nn = n if dim == 2 else 15
        g = etd.unit_box_grid(dim, nn + 1)
        u0 = 0.5 * np.random.default_rng(5).uniform(0.0, 1.0, nn ** dim)
        plan = etd.make_plan(g, 0.01, 1.0, 1.0)
        got = etd.advance(plan, etd.StepperState(0, 0.0, u0), etd.singular(0.1), nsteps=5)
        want = ref_or_oracle().scalar_run(dim, nn, 0.01, 1.0, 1.0, u0, 5, src_kind=5, src_params=(0.1,))[0]
        assert rel_gap(want, got.U) <= STEP_TOL
        bad = u0.copy()
        bad[7] = 1.0
        with pytest.raises(etd.StepperAbort) as ei:
            etd.advance(plan, etd.StepperState(2, 0.02, bad), etd.singular(0.1), nsteps=3)
        assert ei.value.step == -1 and ei.value.t == pytest.approx(0.02)
        u, n_, t = plan.download(0)
        assert n_ == 2 and np.array_equal(u, bad)


@pytest.mark.parametrize("tile", ["0", "1", "2", "3"])
def test_every_tile_class_vs_reference(tile, monkeypatch):
    """Large (8-warp), mid and tiny (4-warp) tile variants of every stage kernel,
    forced on the same small problems, all match the reference."""
    monkeypatch.setenv("ETD_FORCE_TILE", tile)
    R = ref_or_oracle()
    rng = np.random.default_rng(int(tile) + 40)
    g = etd.unit_box_grid(3, 26)
    c0, c1 = rng.uniform(-1, 1, 25 ** 3), rng.uniform(-1, 1, 25 ** 3)
    sp = etd.make_system_plan(g, 0.05, 1e-3, 5e-4, 0.0)
    got = etd.etd2rkds_step_system(sp, etd.SystemState(0, 0.0, c0, c1), etd.fhn_cubic(), nsteps=3)
    wu, wv = R.system_run(3, 25, 0.05, 1e-3, 5e-4, 0.0, c0, c1, 3)[:2]
    assert rel_gap(wu, got.U) <= STEP_TOL and rel_gap(wv, got.V) <= STEP_TOL
    for dim, n in ((2, 57), (3, 19)):
        g = etd.unit_box_grid(dim, n + 1)
        x = rng.uniform(-1, 1, n ** dim)
        p = etd.make_plan(g, 0.01, 0.7, 1.0, scheme=1)
        got = etd.advance(p, etd.StepperState(0, 0.0, x), etd.allen_cahn_cubic(), nsteps=3)
        want = R.scalar_run(dim, n, 0.01, 0.7, 1.0, x, 3, src_kind=1, family=1)[0]
        assert rel_gap(want, got.U) <= STEP_TOL
        for axis in range(dim):
            P, _ = Oracle.spectral_factor(n, 2.0, -1.0)
            t = p.debug_transform(x, axis)
            w = Oracle.contract((n, n, n if dim == 3 else 1), P, x, axis, True)
            assert np.max(np.abs(t - w)) <= 1e-13


@pytest.mark.parametrize("dim,n,steps", [(2, 48, 5), (3, 20, 4), (2, 12, 3)])
def test_exact_exponential_backend_vs_reference(dim, n, steps):
    """BackendKind.ExactExpReference on the device transforms against the
    reference's etd2rkds_reference_step (stepper.cpp:259-295; the reference caps
    it at 64 points per axis, so parity is checked there)."""
    g = etd.unit_box_grid(dim, n + 1)
    u0 = np.random.default_rng(dim + n).uniform(-0.8, 0.8, n ** dim)
    plan = etd.make_plan(g, 0.02, 0.9, 1.0, backend=etd.BackendKind.ExactExpReference)
    got = etd.advance(plan, etd.StepperState(0, 0.0, u0), etd.allen_cahn_cubic(), nsteps=steps)
    if Ref.available():
        want = Ref.scalar_run(dim, n, 0.02, 0.9, 1.0, u0, steps, src_kind=1, backend=3)[0]
        assert rel_gap(want, got.U) <= STEP_TOL
    # exact decay of a sine mode under a zero source (test_stepper.cpp:96-112)
    s = sine_mode(g)
    out = etd.advance(plan, etd.StepperState(0, 0.0, s), etd.DeviceSource(etd.SourceKind.ZERO))
    mu = sum(etd.setup_axis(n, 0.9, 1.0, dim)[1][0] for _ in range(dim))
    assert np.max(np.abs(out.U - np.exp(-0.02 * mu) * s)) <= 1e-12


def test_exact_exponential_backend_beyond_reference_cap():
    """No 64-point cap on the device: a 200^2 exact-exponential run stays consistent
    with the P04 Pade run to the Pade approximation error."""
    n = 200
    g = etd.unit_box_grid(2, n + 1)
    u0 = np.random.default_rng(2).uniform(-0.5, 0.5, n * n)
    ex = etd.advance(etd.make_plan(g, 1e-4, 1.0, 0.0, backend=etd.BackendKind.ExactExpReference),
                     etd.StepperState(0, 0.0, u0), etd.allen_cahn_cubic(), nsteps=5)
    p4 = etd.advance(etd.make_plan(g, 1e-4, 1.0, 0.0, scheme=1), etd.StepperState(0, 0.0, u0),
                     etd.allen_cahn_cubic(), nsteps=5)
    assert np.all(np.isfinite(ex.U)) and rel_gap(ex.U, p4.U) < 1e-2


def test_direct_step_entry_points_and_apply_Q():
    """etd2rkds_step_2d / _3d / etd2rkds_reference_step (stepper.cpp:182-295) and
    StepperPlan::apply_Q (stepper.cpp:106-116) through the mirror."""
    R = ref_or_oracle()
    for dim, n in ((2, 31), (3, 15)):
        g = etd.unit_box_grid(dim, n + 1)
        u0 = np.random.default_rng(40 + dim).uniform(-1, 1, n ** dim)
        plan = etd.make_plan(g, 0.01, 1.0, 1.0)
        step = etd.etd2rkds_step_2d if dim == 2 else etd.etd2rkds_step_3d
        other = etd.etd2rkds_step_3d if dim == 2 else etd.etd2rkds_step_2d
        got = step(plan, etd.StepperState(0, 0.0, u0), etd.allen_cahn_cubic())
        want = R.scalar_run(dim, n, 0.01, 1.0, 1.0, u0, 1, src_kind=1)[0]
        assert got.n == 1 and rel_gap(want, got.U) <= STEP_TOL
        with pytest.raises(etd.ConfigError):
            other(plan, etd.StepperState(0, 0.0, u0), etd.allen_cahn_cubic())
        with pytest.raises(etd.ConfigError):
            etd.etd2rkds_reference_step(plan, etd.StepperState(0, 0.0, u0), etd.allen_cahn_cubic())
        for axis in range(dim):
            q = plan.apply_Q(2, u0, axis)
            assert rel_gap(R.apply_q(dim, n, 0.01, 1.0, 1.0, 0, 2, axis, u0), q) <= 1e-12
        ex = etd.make_plan(g, 0.01, 1.0, 1.0, backend=etd.BackendKind.ExactExpReference)
        a = etd.etd2rkds_reference_step(ex, etd.StepperState(0, 0.0, u0), etd.allen_cahn_cubic())
        b = etd.advance(ex, etd.StepperState(0, 0.0, u0), etd.allen_cahn_cubic())
        assert np.array_equal(a.U, b.U)
