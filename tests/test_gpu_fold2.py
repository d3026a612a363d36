"""GPU: the second-level parity split (etd_kernels.cuh FOLD 5 and
etd_fold2).

On axes with n = 4H - 1, H a multiple of 8 (n = 32m - 1: every BASELINE config),
each forward transform is an HBM-bound stack pass (etd_fold2) followed by two
launches of H-long contractions: the even-mode group (DST-III halves, FOLD 5) and
the odd-mode group (the DST-I of size h - 1 split again, FOLD 4).  The backward
transforms stay first-level, reading the level-2 mode positions.  These tests
run the level-2 path against the reference (oracle/_ref, else the C
restatement), the first-level path (ETD_FOLD2=0) and the dense path
(ETD_DENSE=1) over 2D/3D, scalar and two-species steps, every tile class, the
pipelined host-buffer advance, aborts and the z-slab sharded schedule.
"""
import numpy as np
import pytest

import paper_2601_06849_b200 as etd
from oracle import Oracle, Ref, rel_gap

pytestmark = pytest.mark.gpu

STEP_TOL = 1e-11


def R():
    return Ref if Ref.available() else Oracle


@pytest.fixture(autouse=True)
def force_level2(monkeypatch):
    """The test grids are below the default size threshold (2^18 points): force it."""
    monkeypatch.setenv("ETD_FOLD2", "1")


def plans(make, monkeypatch):
    """(level-2, level-1, dense) plans of the same problem."""
    p2 = make()
    monkeypatch.setenv("ETD_FOLD2", "0")
    p1 = make()
    monkeypatch.setenv("ETD_FOLD2", "1")
    monkeypatch.setenv("ETD_DENSE", "1")
    pd = make()
    monkeypatch.delenv("ETD_DENSE")
    return p2, p1, pd


@pytest.mark.parametrize("dim,n", [(2, 31), (2, 63), (2, 127), (3, 31), (3, 63)])
def test_fold2_apply_q_and_scalar_steps(dim, n, monkeypatch):
    g = etd.unit_box_grid(dim, n + 1)
    x = np.random.default_rng(n + dim).uniform(-0.5, 0.5, n ** dim)
    tau, kappa, q = 0.02, 0.7, 1.0
    p2, p1, pd = plans(lambda: etd.make_plan(g, tau, kappa, q, source=etd.allen_cahn_cubic()), monkeypatch)
    assert p2.fold_level() == (2,) * dim and p1.fold_level() == (1,) * dim and pd.fold_level() == (0,) * dim
    for axis in range(dim):
        for ell in (1, 2, 3):
            a = p2.apply_Q(ell, x, axis)
            want = R().apply_q(dim, n, tau, kappa, q, 0, ell, axis, x)
            assert np.max(np.abs(a - want)) <= 1e-12, (axis, ell)
            assert np.max(np.abs(a - pd.apply_Q(ell, x, axis))) <= 1e-13, (axis, ell)
    s0 = etd.StepperState(0, 0.0, x)
    a = etd.advance(p2, s0, etd.allen_cahn_cubic(), nsteps=4)
    b = etd.advance(p1, s0, etd.allen_cahn_cubic(), nsteps=4)
    want = R().scalar_run(dim, n, tau, kappa, q, x, 4, src_kind=1)[0]
    assert rel_gap(want, a.U) <= STEP_TOL
    assert rel_gap(b.U, a.U) <= 1e-13
    assert a.n == 4 and abs(a.t - 4 * tau) < 1e-15


@pytest.mark.parametrize("n", [31, 63])
def test_fold2_system_3d_vs_reference_and_level1(n, monkeypatch):
    g = etd.unit_box_grid(3, n + 1)
    rng = np.random.default_rng(n)
    u0, v0 = rng.uniform(-1, 1, n ** 3), rng.uniform(-0.5, 0.5, n ** 3)
    p2, p1, _ = plans(lambda: etd.make_system_plan(g, 0.05, 1e-3, 5e-4, 0.0), monkeypatch)
    st = etd.SystemState(0, 0.0, u0, v0)
    a = etd.etd2rkds_step_system(p2, st, etd.fhn_cubic(), nsteps=3)
    b = etd.etd2rkds_step_system(p1, st, etd.fhn_cubic(), nsteps=3)
    wu, wv = R().system_run(3, n, 0.05, 1e-3, 5e-4, 0.0, u0, v0, 3)[:2]
    assert rel_gap(wu, a.U) <= STEP_TOL and rel_gap(wv, a.V) <= STEP_TOL
    assert rel_gap(b.U, a.U) <= 1e-13 and rel_gap(b.V, a.V) <= 1e-13


def test_fold2_config_physics_2d_system(monkeypatch):
    n = 63
    g = etd.unit_box_grid(2, n + 1)
    rng = np.random.default_rng(5)
    u0, v0 = rng.uniform(-1, 1, n * n), rng.uniform(-0.5, 0.5, n * n)
    p2 = etd.make_system_plan(g, 0.05, 1e-3, 5e-4, 0.0)
    assert p2.fold_level() == (2, 2)
    a = etd.etd2rkds_step_system(p2, etd.SystemState(0, 0.0, u0, v0), etd.fhn_cubic(), nsteps=3)
    wu, wv = R().system_run(2, n, 0.05, 1e-3, 5e-4, 0.0, u0, v0, 3)[:2]
    assert rel_gap(wu, a.U) <= STEP_TOL and rel_gap(wv, a.V) <= STEP_TOL


@pytest.mark.parametrize("tile", ["0", "1", "2", "3"])
def test_fold2_every_tile_class(tile, monkeypatch):
    monkeypatch.setenv("ETD_FORCE_TILE", tile)
    n = 63
    g = etd.unit_box_grid(3, n + 1)
    rng = np.random.default_rng(int(tile) + 90)
    u0, v0 = rng.uniform(-1, 1, n ** 3), rng.uniform(-1, 1, n ** 3)
    sp = etd.make_system_plan(g, 0.05, 1e-3, 5e-4, 0.0)
    assert sp.fold_level() == (2, 2, 2)
    got = etd.etd2rkds_step_system(sp, etd.SystemState(0, 0.0, u0, v0), etd.fhn_cubic(), nsteps=2)
    wu, wv = R().system_run(3, n, 0.05, 1e-3, 5e-4, 0.0, u0, v0, 2)[:2]
    assert rel_gap(wu, got.U) <= STEP_TOL and rel_gap(wv, got.V) <= STEP_TOL


def test_fold2_pipelined_advance_equals_resident_steps():
    from paper_2601_06849_b200 import configs
    cfg = configs.CONFIGS[4]
    n = 255
    ics = configs.initial_state(cfg, n)
    plan = configs.make_plan(cfg, n)
    assert plan.fold_level() == (2, 2, 2)
    st = etd.etd2rkds_step_system(plan, etd.SystemState(0, 0.0, *ics), cfg.source, nsteps=2)  # host buffers
    plan.upload(0, ics[0])
    plan.upload(1, ics[1])
    plan.step(2)
    u, nn, _ = plan.download(0)
    v, _, _ = plan.download(1)
    assert nn == 2
    assert np.array_equal(u, st.U) and np.array_equal(v, st.V)


def test_fold2_abort_keeps_input_state():
    """test_stepper.cpp:304-321 on the level-2 schedule: the input state's t and n."""
    n = 31
    g = etd.unit_box_grid(2, n + 1)
    plan = etd.make_plan(g, 0.01, 1.0, 1.0)
    assert plan.fold_level() == (2, 2)
    u0 = np.random.default_rng(7).uniform(-0.5, 0.5, n * n)
    with pytest.raises(etd.StepperAbort) as ei:
        etd.advance(plan, etd.StepperState(4, 0.25, u0), etd.DeviceSource(etd.SourceKind.NAN_PROBE))
    assert ei.value.t == pytest.approx(0.25) and ei.value.step == 4
    u, nn, t = plan.download(0)
    assert nn == 4 and np.array_equal(u, u0)


@pytest.mark.parametrize("G", [2, 3])
def test_fold2_sharded_virtual_ranks_bitwise(G):
    from test_gpu_sharded import run_sharded
    n = 63
    grid = etd.unit_box_grid(3, n + 1)
    rng = np.random.default_rng(G)
    u0, v0 = rng.uniform(-1, 1, n ** 3), rng.uniform(-0.5, 0.5, n ** 3)
    f = etd.fhn_cubic()
    make = lambda **kw: etd.SystemPlan(grid, 0.05, 1e-3, 5e-4, 0.0, source=f, **kw)
    single = make()
    assert single.fold_level() == (2, 2, 2)
    want = etd.etd2rkds_step_system(single, etd.SystemState(0, 0.0, u0, v0), f, nsteps=2)
    (u, v), nn, _ = run_sharded(make, G, [u0, v0], 2, grid, f)
    assert nn == 2
    assert np.array_equal(u, want.U) and np.array_equal(v, want.V)


@pytest.mark.parametrize("G,chunks", [(2, "40"), (3, "13")])
def test_fold2_sharded_empty_chunks_bitwise(G, chunks, monkeypatch):
    """More z-stage chunks than a rank has y rows (ETD_ZCHUNKS > rows per rank) with
    the level-2 split forced and two species: empty chunks must pad the op list with
    exactly as many no-ops as a populated chunk emits (source + 4 + 4 launches +
    unfold with pair launches), or the virtual ranks' op lists misalign."""
    from test_gpu_sharded import run_sharded
    monkeypatch.setenv("ETD_FOLD2", "1")
    monkeypatch.setenv("ETD_ZCHUNKS", chunks)
    n = 31
    grid = etd.unit_box_grid(3, n + 1)
    rng = np.random.default_rng(10 + G)
    u0, v0 = rng.uniform(-1, 1, n ** 3), rng.uniform(-0.5, 0.5, n ** 3)
    f = etd.fhn_cubic()
    make = lambda **kw: etd.SystemPlan(grid, 0.05, 1e-3, 5e-4, 0.0, source=f, **kw)
    single = make()
    assert single.fold_level() == (2, 2, 2)
    want = etd.etd2rkds_step_system(single, etd.SystemState(0, 0.0, u0, v0), f, nsteps=2)
    (u, v), nn, _ = run_sharded(make, G, [u0, v0], 2, grid, f)
    assert nn == 2
    assert np.array_equal(u, want.U) and np.array_equal(v, want.V)


@pytest.mark.parametrize("dim", [2, 3])
def test_fold2_pair_launches_bitwise_equal(dim, monkeypatch):
    """Every S = 4 transform launch runs as two S = 2 launches by default (fields
    (0,1), (2,3); the mix pairs each species' (w1, w2)); ETD_PAIRS=0 keeps one S = 4
    launch.  The same per-element contraction order, so the step is bitwise equal."""
    n = 63
    g = etd.unit_box_grid(dim, n + 1)
    rng = np.random.default_rng(40 + dim)
    u0, v0 = rng.uniform(-1, 1, n ** dim), rng.uniform(-0.5, 0.5, n ** dim)
    st = etd.SystemState(0, 0.0, u0, v0)
    monkeypatch.setenv("ETD_PAIRS", "0")
    a = etd.etd2rkds_step_system(etd.make_system_plan(g, 0.05, 1e-3, 5e-4, 0.0), st, etd.fhn_cubic(), nsteps=2)
    monkeypatch.delenv("ETD_PAIRS")
    pp = etd.make_system_plan(g, 0.05, 1e-3, 5e-4, 0.0)
    assert any(s["name"].endswith("_b") for s in pp.stage_stats())
    b = etd.etd2rkds_step_system(pp, st, etd.fhn_cubic(), nsteps=2)
    assert np.array_equal(a.U, b.U) and np.array_equal(a.V, b.V)


@pytest.mark.parametrize("shape", [(63, 95, 31), (95, 31, 63), (31, 63, 127)])
def test_fold2_non_cubic_system_vs_dense(shape, monkeypatch):
    """Different H per axis (8, 16, 24, 32): the fused z unfold + y stack pass and the
    x / y stack passes index each axis with its own H.  Compared with the dense path
    (itself pinned to the reference on non-cubic grids, test_gpu_parity.py)."""
    g = etd.build_grid(3, [(0, 1)] * 3, [s + 1 for s in shape])
    N = int(np.prod(shape))
    rng = np.random.default_rng(sum(shape))
    u0, v0 = rng.uniform(-1, 1, N), rng.uniform(-0.5, 0.5, N)
    p = etd.make_system_plan(g, 0.05, 1e-3, 5e-4, 0.0)
    assert p.fold_level() == (2, 2, 2)
    # fused backward (default): z_back then the y stack pass; r01 path: z unfold + y stack in one pass
    assert any(s["name"] in ("fold_y_fwd", "z_back_y_stack") for s in p.stage_stats())
    got = etd.etd2rkds_step_system(p, etd.SystemState(0, 0.0, u0, v0), etd.fhn_cubic(), nsteps=3)
    monkeypatch.setenv("ETD_DENSE", "1")
    pd = etd.make_system_plan(g, 0.05, 1e-3, 5e-4, 0.0)
    d = etd.etd2rkds_step_system(pd, etd.SystemState(0, 0.0, u0, v0), etd.fhn_cubic(), nsteps=3)
    assert rel_gap(d.U, got.U) <= 1e-13 and rel_gap(d.V, got.V) <= 1e-13


@pytest.mark.parametrize("back6", ["1", "0"])
@pytest.mark.parametrize("shape", [(127, 95, 63), (95, 63, 1)])
def test_fold2_pipelined_advance_ragged_chunks_bitwise(shape, back6, monkeypatch):
    """etd_advance (column-chunked z / y stages, row-chunked x stage) on the level-2
    schedule equals upload + etd_step + download bitwise, 3D and 2D; fused backward
    launches (default) and the round-1 two-launch + unfold path (ETD_BACK6=0)."""
    monkeypatch.setenv("ETD_BACK6", back6)
    nx, ny, nz = shape
    dim = 3 if nz > 1 else 2
    g = etd.build_grid(dim, [(0, 1)] * dim, [s + 1 for s in shape[:dim]])
    N = nx * ny * nz
    rng = np.random.default_rng(N)
    u0, v0 = rng.uniform(-1, 1, N), rng.uniform(-0.5, 0.5, N)
    f = etd.fhn_cubic()
    plan = etd.make_system_plan(g, 0.05, 1e-3, 5e-4, 0.0)
    assert plan.fold_level() == (2,) * dim
    st = etd.etd2rkds_step_system(plan, etd.SystemState(0, 0.0, u0, v0), f, nsteps=2)
    plan.upload(0, u0)
    plan.upload(1, v0)
    plan.step(2)
    assert np.array_equal(plan.download(0)[0], st.U) and np.array_equal(plan.download(1)[0], st.V)


@pytest.mark.parametrize("dim,n", [(3, 255), (2, 1023)])
def test_fused_backward_bitwise_equals_two_launch_path(dim, n, monkeypatch):
    """The fused level-2 backward (etd_back6) accumulates every output with the same
    DMMA sequence as the two launches + unfold pass it replaces (G6 holds GO / GE's
    rows, tests/test_fold_cpu.py), so whole steps are bitwise equal; at n = 255 the
    k loop refills the 2-stage ring (the proxy-fenced release, etd_kernels.cuh)."""
    g = etd.unit_box_grid(dim, n + 1)
    rng = np.random.default_rng(n + dim)
    N = n ** dim
    u0, v0 = rng.uniform(-1, 1, N), rng.uniform(-0.5, 0.5, N)
    out = []
    for b6 in ("1", "0"):
        monkeypatch.setenv("ETD_BACK6", b6)
        p = etd.make_system_plan(g, 0.05, 1e-3, 5e-4, 0.0, source=etd.fhn_cubic())
        assert p.fold_level() == (2,) * dim
        p.upload(0, u0)
        p.upload(1, v0)
        p.step(3)
        out.append((p.download(0)[0], p.download(1)[0]))
        p.close()
    assert np.array_equal(out[0][0], out[1][0]) and np.array_equal(out[0][1], out[1][1])
