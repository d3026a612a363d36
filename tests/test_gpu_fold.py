"""GPU: the parity-split transforms (etd_kernels.cuh FOLD 1-4).

Every axis whose half extent h = (n+1)/2 is a multiple of 8 (n = 16m-1 or 16m,
all five BASELINE configs) runs its eigenbasis transforms as two h x h dense
contractions over the symmetric / antisymmetric halves of each pencil.  These
tests run the folded path against the reference (oracle/_ref, else the C
restatement) and against the dense path of the same plan (ETD_DENSE=1), over
odd and even n, mixed folded / dense axes, every tile class, every epilogue and
source kind, the pipelined host-buffer advance, aborts and the z-slab sharded
schedule.  Tolerances as in test_gpu_parity.py.
"""
import numpy as np
import pytest

import paper_2601_06849_b200 as etd
from oracle import Oracle, Ref, rel_gap

pytestmark = pytest.mark.gpu

STEP_TOL = 1e-11


def R():
    return Ref if Ref.available() else Oracle


def folded(n):
    return ((n + 1) // 2) % 8 == 0


@pytest.mark.parametrize("dim,n", [(2, 15), (2, 16), (2, 63), (2, 127), (3, 15), (3, 31), (3, 32), (3, 47)])
def test_fold_apply_q_and_steps_vs_dense_and_reference(dim, n, monkeypatch):
    assert folded(n)
    g = etd.unit_box_grid(dim, n + 1)
    x = np.random.default_rng(n + dim).uniform(-0.5, 0.5, n ** dim)
    tau, kappa, q = 0.02, 0.7, 1.0
    pf = etd.make_plan(g, tau, kappa, q, source=etd.allen_cahn_cubic())
    monkeypatch.setenv("ETD_DENSE", "1")
    pd = etd.make_plan(g, tau, kappa, q, source=etd.allen_cahn_cubic())
    monkeypatch.delenv("ETD_DENSE")
    for axis in range(dim):
        for ell in (1, 2, 3):
            a = pf.apply_Q(ell, x, axis)
            b = pd.apply_Q(ell, x, axis)
            want = R().apply_q(dim, n, tau, kappa, q, 0, ell, axis, x)
            assert np.max(np.abs(a - want)) <= 1e-12, (axis, ell)
            assert np.max(np.abs(a - b)) <= 1e-13, (axis, ell)
    a = etd.advance(pf, etd.StepperState(0, 0.0, x), etd.allen_cahn_cubic(), nsteps=4)
    b = etd.advance(pd, etd.StepperState(0, 0.0, x), etd.allen_cahn_cubic(), nsteps=4)
    want = R().scalar_run(dim, n, tau, kappa, q, x, 4, src_kind=1)[0]
    assert rel_gap(want, a.U) <= STEP_TOL
    assert rel_gap(b.U, a.U) <= 1e-13


def test_fold_mixed_axes_system_equals_dense(monkeypatch):
    """x and z folded (47, 31), y dense (25): every stage follows its own axis."""
    shape = (47, 25, 31)
    g = etd.build_grid(3, [(0, 1)] * 3, [s + 1 for s in shape])
    N = int(np.prod(shape))
    rng = np.random.default_rng(7)
    u0, v0 = rng.uniform(-1, 1, N), rng.uniform(-0.5, 0.5, N)
    plan = etd.make_system_plan(g, 0.05, 1e-3, 5e-4, 0.0)
    got = etd.etd2rkds_step_system(plan, etd.SystemState(0, 0.0, u0, v0), etd.fhn_cubic(), nsteps=3)
    monkeypatch.setenv("ETD_DENSE", "1")
    pd = etd.make_system_plan(g, 0.05, 1e-3, 5e-4, 0.0)
    dense = etd.etd2rkds_step_system(pd, etd.SystemState(0, 0.0, u0, v0), etd.fhn_cubic(), nsteps=3)
    assert rel_gap(dense.U, got.U) <= 1e-13 and rel_gap(dense.V, got.V) <= 1e-13
    assert plan.parity_split() == (True, False, True) and pd.parity_split() == (False, False, False)


@pytest.mark.parametrize("tile", ["0", "1", "2", "3"])
def test_fold_every_tile_class_vs_reference(tile, monkeypatch):
    monkeypatch.setenv("ETD_FORCE_TILE", tile)
    rng = np.random.default_rng(int(tile) + 70)
    n = 31
    g = etd.unit_box_grid(3, n + 1)
    c0, c1 = rng.uniform(-1, 1, n ** 3), rng.uniform(-1, 1, n ** 3)
    sp = etd.make_system_plan(g, 0.05, 1e-3, 5e-4, 0.0)
    got = etd.etd2rkds_step_system(sp, etd.SystemState(0, 0.0, c0, c1), etd.fhn_cubic(), nsteps=3)
    wu, wv = R().system_run(3, n, 0.05, 1e-3, 5e-4, 0.0, c0, c1, 3)[:2]
    assert rel_gap(wu, got.U) <= STEP_TOL and rel_gap(wv, got.V) <= STEP_TOL
    for dim, n in ((2, 63), (3, 15), (2, 48)):
        g = etd.unit_box_grid(dim, n + 1)
        x = rng.uniform(-1, 1, n ** dim)
        p = etd.make_plan(g, 0.01, 0.7, 1.0, scheme=1)
        got = etd.advance(p, etd.StepperState(0, 0.0, x), etd.allen_cahn_cubic(), nsteps=3)
        want = R().scalar_run(dim, n, 0.01, 0.7, 1.0, x, 3, src_kind=1, family=1)[0]
        assert rel_gap(want, got.U) <= STEP_TOL
        for axis in range(dim):
            a = p.apply_Q(2, x, axis)
            want = R().apply_q(dim, n, 0.01, 0.7, 1.0, 1, 2, axis, x)
            assert np.max(np.abs(a - want)) <= 1e-12


@pytest.mark.parametrize("dim,n", [(2, 47), (3, 31)])
def test_fold_catalogue_sources_vs_reference(dim, n):
    """Manufactured Allen-Cahn (position dependent: sin tables at mirrored x in the
    folded epilogue) and the singular source with its domain guard."""
    g = etd.unit_box_grid(dim, n + 1)
    src = etd.allen_cahn_manufactured(dim, 1.0, 1.0)
    u0 = np.random.default_rng(21).uniform(0.0, 0.8, n ** dim)
    plan = etd.make_plan(g, 0.01, 1.0, 0.0)
    got = etd.advance(plan, etd.StepperState(3, 0.03, u0), src, nsteps=4)
    want = R().scalar_run(dim, n, 0.01, 1.0, 0.0, u0, 4, src_kind=4, src_params=src.params8(), n0=3, t0=0.03)[0]
    assert rel_gap(want, got.U) <= STEP_TOL
    u1 = 0.5 * np.random.default_rng(5).uniform(0.0, 1.0, n ** dim)
    plan = etd.make_plan(g, 0.01, 1.0, 1.0)
    got = etd.advance(plan, etd.StepperState(0, 0.0, u1), etd.singular(0.1), nsteps=4)
    want = R().scalar_run(dim, n, 0.01, 1.0, 1.0, u1, 4, src_kind=5, src_params=(0.1,))[0]
    assert rel_gap(want, got.U) <= STEP_TOL
    bad = u1.copy()
    bad[n - 1] = 1.0   # last x of the first row: a mirrored column of the folded epilogue
    with pytest.raises(etd.StepperAbort) as ei:
        etd.advance(plan, etd.StepperState(2, 0.02, bad), etd.singular(0.1), nsteps=3)
    assert ei.value.step == -1 and ei.value.t == pytest.approx(0.02)


def test_fold_nonfinite_aborts_keep_input_state():
    n = 31
    g = etd.unit_box_grid(3, n + 1)
    plan = etd.make_plan(g, 0.01, 1.0, 1.0)
    u0 = np.random.default_rng(3).uniform(-0.5, 0.5, n ** 3)
    with pytest.raises(etd.StepperAbort) as ei:
        etd.advance(plan, etd.StepperState(9, 0.09, u0), etd.DeviceSource(etd.SourceKind.NAN_PROBE), nsteps=3)
    assert ei.value.step == 9 and ei.value.t == pytest.approx(0.09)
    u, nn, t = plan.download(0)
    assert nn == 9 and np.array_equal(u, u0)


def test_fold_pipelined_advance_equals_device_resident_steps():
    grid = etd.build_grid(3, [(0, 1)] * 3, [48, 32, 64])   # 47 x 31 x 63 interior: every axis folded
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
        assert a.n == n == 2 + steps


@pytest.mark.parametrize("G", [2, 3, 4])
def test_fold_sharded_equals_single_gpu(G):
    from test_gpu_sharded import run_sharded
    grid = etd.build_grid(3, [(0, 1)] * 3, [32, 48, 48])   # 31 x 47 x 47 interior, uneven slabs
    nx, ny, nz = grid.interior_shape()
    rng = np.random.default_rng(G + 30)
    u0, v0 = rng.uniform(-1, 1, nx * ny * nz), rng.uniform(-0.5, 0.5, nx * ny * nz)
    f = etd.fhn_cubic()
    make = lambda **kw: etd.SystemPlan(grid, 0.05, 1e-3, 5e-4, 0.0, source=f, **kw)
    ref = etd.etd2rkds_step_system(make(), etd.SystemState(0, 0.0, u0, v0), f, nsteps=3)
    (u, v), n, t = run_sharded(make, G, [u0, v0], 3, grid, f)
    assert n == 3 and np.array_equal(u, ref.U) and np.array_equal(v, ref.V)


def test_fold_halves_the_transform_flops(monkeypatch):
    """Stage FLOPs reported per launch: the folded transform executes 2 (2h) h / n
    per point against 2 n dense."""
    monkeypatch.setenv("ETD_FOLD2", "1")   # below the default size threshold
    monkeypatch.setenv("ETD_PAIRS", "0")
    n = 63
    g = etd.unit_box_grid(3, n + 1)
    p = etd.make_plan(g, 0.01, 1.0, 1.0, source=etd.allen_cahn_cubic())
    st = {s["name"]: s for s in p.stage_stats()}
    pts = n ** 3
    h = (n + 1) // 2
    H = h // 2
    # second level: each of the two forward launches 2 (2H) H / n per point
    assert p.fold_level() == (2, 2, 2)
    for nm in ("z_fwd_even", "z_fwd_odd"):
        assert st[nm]["flops_per_launch"] == pytest.approx(2.0 * 2 * H * H / n * pts * 2)
        assert st[nm]["dense_flops_per_launch"] == pytest.approx(0.5 * 2.0 * n * pts * 2)
    # the fused backward (§4c): one launch of all four quarters, 2 (4H) H / n per point
    # (n = 63: 4H = 64 rows, already whole 64-row block pairs)
    # (y/z: one launch per field of the [U, fU] stack)
    for nm in ("z_back_a", "z_back_b"):
        assert st[nm]["flops_per_launch"] == pytest.approx(2.0 * 4 * H * H / n * pts)
        assert st[nm]["dense_flops_per_launch"] == pytest.approx(2.0 * n * pts)
    # the y stack pass (HBM-bound, no FLOPs counted)
    assert st["fold_y_fwd"]["flops_per_launch"] == 0
    # the round-1 backward: two launches + the fused z unfold / y stack pass
    monkeypatch.setenv("ETD_BACK6", "0")
    st = {s["name"]: s for s in etd.make_plan(g, 0.01, 1.0, 1.0, source=etd.allen_cahn_cubic()).stage_stats()}
    for nm in ("z_back_o", "z_back_e"):
        assert st[nm]["flops_per_launch"] == pytest.approx(2.0 * 2 * H * H / n * pts * 2)
    assert st["z_back_y_stack"]["flops_per_launch"] == 0 and st["y_back"]["flops_per_launch"] == 0


@pytest.mark.parametrize("shape", [(127, 31, 47), (200, 41, 1), (255, 63, 1), (130, 20, 33)])
def test_pipelined_advance_x_column_chunks_equal_device_resident_steps(shape):
    """etd_advance uploads in x-column ranges and runs the first step's source and
    z / y stages per range, then the last step's x stage in row chunks with the
    download behind it: bitwise equal to upload + etd_step + download (2D and 3D,
    folded and dense axes, several column chunks, ragged last chunk)."""
    nx, ny, nz = shape
    dim = 3 if nz > 1 else 2
    grid = etd.build_grid(dim, [(0, 1)] * dim, [s + 1 for s in shape[:dim]])
    N = nx * ny * nz
    rng = np.random.default_rng(N)
    u0, v0 = rng.uniform(-1, 1, N), rng.uniform(-0.5, 0.5, N)
    f = etd.fhn_cubic()
    for steps in (1, 2):
        plan = etd.make_system_plan(grid, 0.05, 1e-3, 5e-4, 0.0)
        a = etd.etd2rkds_step_system(plan, etd.SystemState(4, 0.2, u0, v0), f, nsteps=steps)
        plan2 = etd.make_system_plan(grid, 0.05, 1e-3, 5e-4, 0.0, source=f)
        plan2.upload(0, u0, 4, 0.2)
        plan2.upload(1, v0, 4, 0.2)
        plan2.step(steps)
        bu, n, t = plan2.download(0)
        bv, _, _ = plan2.download(1)
        assert np.array_equal(a.U, bu) and np.array_equal(a.V, bv), (shape, steps)
        assert a.n == n == 4 + steps
    g1 = etd.make_plan(grid, 0.01, 1.0, 1.0)
    s1 = etd.advance(g1, etd.StepperState(0, 0.0, u0), etd.allen_cahn_cubic(), nsteps=1)
    g2 = etd.make_plan(grid, 0.01, 1.0, 1.0, source=etd.allen_cahn_cubic())
    g2.upload(0, u0)
    g2.step(1)
    assert np.array_equal(s1.U, g2.download(0)[0])
