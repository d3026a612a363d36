"""GPU: ETRD field snapshots straight from/to device state, in the reference's
own format (field.cpp:32-81): files written by the device plan load in the
reference's load_field and vice versa; restart from a snapshot continues the
run bitwise."""
import os

import numpy as np
import pytest

import paper_2601_06849_b200 as etd
from oracle import Ref

pytestmark = pytest.mark.gpu


def test_snapshot_roundtrip_and_reference_format(tmp_path):
    g = etd.build_grid(3, [(0, 1)] * 3, [20, 18, 16])
    nx, ny, nz = g.interior_shape()
    u0 = np.random.default_rng(0).uniform(-1, 1, nx * ny * nz)
    plan = etd.make_plan(g, 0.01, 1.0, 1.0)
    plan.upload(0, u0, 0, 0.0)
    plan.step(3)
    u3, n3, t3 = plan.download(0)
    path = str(tmp_path / "s.etrd")
    plan.save_snapshot(0, path)
    if Ref.available():
        data, shape, t = Ref.load_field(path, nx * ny * nz)
        assert shape == (3, nx, ny, nz) and t == t3 and np.array_equal(data, u3)
        path2 = str(tmp_path / "r.etrd")
        Ref.save_field((nx, ny, nz), u0, 0.125, path2)
        plan.load_snapshot(0, path2)
        u, n, t = plan.download(0)
        assert np.array_equal(u, u0) and t == 0.125 and n == int(np.floor(0.125 / 0.01 + 0.5))  # llround
    # restart: 3 steps, snapshot, fresh plan, 2 more == 5 straight steps
    fresh = etd.make_plan(g, 0.01, 1.0, 1.0)
    fresh.load_snapshot(0, path)
    fresh.step(2)
    a, na, ta = fresh.download(0)
    plan.upload(0, u0, 0, 0.0)
    plan.step(5)
    b, nb, tb = plan.download(0)
    assert np.array_equal(a, b) and na == nb == 5 and ta == pytest.approx(tb)


def test_snapshot_guards(tmp_path):
    g = etd.unit_box_grid(2, 10)
    plan = etd.make_plan(g, 0.01, 1.0, 1.0)
    bad = np.zeros(81)
    bad[5] = np.nan
    plan.upload(0, bad)
    with pytest.raises(etd.NumericsError):
        plan.save_snapshot(0, str(tmp_path / "x.etrd"))
    plan.upload(0, np.ones(81))
    plan.save_snapshot(0, str(tmp_path / "ok.etrd"))
    other = etd.make_plan(etd.unit_box_grid(2, 12), 0.01, 1.0, 1.0)
    with pytest.raises(etd.ConfigError):
        other.load_snapshot(0, str(tmp_path / "ok.etrd"))
    (tmp_path / "junk.etrd").write_bytes(b"NOPE" + b"\0" * 64)
    with pytest.raises(etd.ConfigError):
        plan.load_snapshot(0, str(tmp_path / "junk.etrd"))


def test_failed_load_leaves_state_untouched(tmp_path):
    """A truncated or non-finite snapshot raises and leaves the device state, n and
    t as they were (the reference's load_field has no side effects on failure)."""
    g = etd.unit_box_grid(3, 12)
    plan = etd.make_plan(g, 0.01, 1.0, 1.0)
    u0 = np.random.default_rng(3).uniform(-1, 1, 11 ** 3)
    plan.upload(0, u0, 4, 0.04)
    good = str(tmp_path / "good.etrd")
    plan.save_snapshot(0, good)
    raw = open(good, "rb").read()
    trunc = str(tmp_path / "trunc.etrd")
    open(trunc, "wb").write(raw[: len(raw) - 8 * 200])
    nanf = str(tmp_path / "nan.etrd")
    body = np.frombuffer(raw[32:], dtype=np.float64).copy()
    body[-1] = np.nan
    open(nanf, "wb").write(raw[:32] + body.tobytes())
    plan.upload(0, 0.5 * u0, 9, 0.09)
    for path, exc in ((trunc, etd.ConfigError), (nanf, etd.NumericsError)):
        with pytest.raises(exc):
            plan.load_snapshot(0, path)
        u, n, t = plan.download(0)
        assert np.array_equal(u, 0.5 * u0) and n == 9 and t == pytest.approx(0.09)
