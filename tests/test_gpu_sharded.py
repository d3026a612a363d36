"""GPU: the z-slab sharded schedule (partition, pack, chunked exchanges, z stage
on y-row chunks, exchanges back, unpack, global abort agreement) run as G virtual
ranks on ONE device via etd_group_step.  Every per-pencil contraction is the
same arithmetic as on the unsharded plan, so results must be bitwise equal."""
import numpy as np
import pytest

import paper_2601_06849_b200 as etd
from oracle import Ref, Oracle, rel_gap

pytestmark = pytest.mark.gpu


def run_sharded(make, G, fields, nsteps, grid, f):
    nx, ny, nz = grid.interior_shape()
    plans = [make(world_size=G, rank=r) for r in range(G)]
    for p in plans:
        z0, z1 = p.slab
        for s, a in enumerate(fields):
            p.upload(s, a.reshape(nz, ny, nx)[z0:z1], 0, 0.0)
        p.set_source(f)
    etd.group_step(plans, nsteps)
    outs = []
    for s in range(len(fields)):
        outs.append(np.concatenate([p.download(s)[0].reshape(-1, ny, nx) for p in plans]).reshape(-1))
    n, t = plans[0].download(0)[1:]
    for p in plans:
        p.close()
    return outs, n, t


@pytest.mark.parametrize("G,chunks", [(2, None), (3, None), (4, None), (2, "1"), (3, "3"), (4, "9")])
def test_sharded_system_equals_single_gpu(G, chunks, monkeypatch):
    """Default 4 z-stage chunks, plus 1, 3 and more chunks than a rank has rows (empty chunks)."""
    if chunks:
        monkeypatch.setenv("ETD_ZCHUNKS", chunks)
    grid = etd.build_grid(3, [(0, 1)] * 3, [38, 30, 24])   # 37 x 29 x 23 interior, uneven splits
    nx, ny, nz = grid.interior_shape()
    rng = np.random.default_rng(G)
    u0, v0 = rng.uniform(-1, 1, nx * ny * nz), rng.uniform(-0.5, 0.5, nx * ny * nz)
    f = etd.fhn_cubic()
    make = lambda **kw: etd.SystemPlan(grid, 0.05, 1e-3, 5e-4, 0.0, source=f, **kw)
    single = make()
    ref = etd.etd2rkds_step_system(single, etd.SystemState(0, 0.0, u0, v0), f, nsteps=4)
    (u, v), n, t = run_sharded(make, G, [u0, v0], 4, grid, f)
    assert n == 4 and t == pytest.approx(0.2)
    assert np.array_equal(u, ref.U) and np.array_equal(v, ref.V)


@pytest.mark.parametrize("G", [2, 5])
def test_sharded_scalar_p04_equals_single_and_reference(G):
    n = 21
    grid = etd.unit_box_grid(3, n + 1)
    u0 = np.random.default_rng(9).uniform(-1, 1, n ** 3)
    f = etd.allen_cahn_cubic()
    make = lambda **kw: etd.StepperPlan(grid, 0.01, 0.3, 1.0, family=1, source=f, **kw)
    single = etd.advance(make(), etd.StepperState(0, 0.0, u0), f, nsteps=3)
    (u,), _, _ = run_sharded(make, G, [u0], 3, grid, f)
    assert np.array_equal(u, single.U)
    R = Ref if Ref.available() else Oracle
    want = R.scalar_run(3, n, 0.01, 0.3, 1.0, u0, 3, src_kind=1, family=1)[0]
    assert rel_gap(want, u) <= 1e-11


def test_sharded_abort_is_global():
    """A non-finite source on one rank aborts the step on every rank, keeping the
    input state and reporting its (t, n) (test_stepper.cpp:304-321)."""
    grid = etd.unit_box_grid(3, 12)
    G = 3
    u0 = np.random.default_rng(1).uniform(-0.5, 0.5, 11 ** 3)
    plans = [etd.StepperPlan(grid, 0.01, 1.0, 1.0, world_size=G, rank=r) for r in range(G)]
    for p in plans:
        z0, z1 = p.slab
        p.upload(0, u0.reshape(11, 11, 11)[z0:z1], 7, 0.35)
        p.set_source(etd.DeviceSource(etd.SourceKind.NAN_PROBE))
    with pytest.raises(etd.StepperAbort) as ei:
        etd.group_step(plans, 2)
    assert ei.value.step == 7 and ei.value.t == pytest.approx(0.35)
    for p in plans:
        u, n, t = p.download(0)
        z0, z1 = p.slab
        assert n == 7 and np.array_equal(u, u0.reshape(11, 11, 11)[z0:z1].reshape(-1))


def test_sharded_position_dependent_source_equals_single_gpu():
    """The manufactured Allen-Cahn source reads sin(pi x) tables at GLOBAL (y, z)
    indices: on y-row blocks (z stage) and z-slabs (x/y stages) the offsets must
    line up exactly with the unsharded plan."""
    grid = etd.build_grid(3, [(0, 1)] * 3, [30, 27, 25])
    nx, ny, nz = grid.interior_shape()
    u0 = np.random.default_rng(4).uniform(0.0, 0.8, nx * ny * nz)
    f = etd.allen_cahn_manufactured(3)
    make = lambda **kw: etd.StepperPlan(grid, 0.01, 1.0, 0.0, source=f, **kw)
    single = etd.advance(make(), etd.StepperState(0, 0.0, u0), f, nsteps=3)
    for G in (2, 3):
        (u,), n, t = run_sharded(make, G, [u0], 3, grid, f)
        assert np.array_equal(u, single.U)
