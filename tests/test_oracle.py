"""CPU: the oracle restatement (oracle/etd_oracle.c) pinned to the reference's own
outputs (tests/golden/*.npz made by oracle/_ref = the unmodified etdrd core), and
to the live reference build when it is present."""
import glob
import os

import numpy as np
import pytest

from oracle import Oracle, Ref, rel_gap

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CASES = sorted(p for p in glob.glob(os.path.join(GOLD, "*.npz")) if not p.endswith("setup.npz"))


def load(p):
    z = np.load(p)
    return {k: z[k] for k in z.files}


@pytest.mark.parametrize("path", CASES, ids=[os.path.basename(p)[:-4] for p in CASES])
def test_oracle_matches_reference_golden(path):
    c = load(path)
    dim, n, steps, fam = int(c["dim"]), int(c["n"]), int(c["steps"]), int(c["family"])
    if str(c["kind"]) == "scalar":
        u, nn, tt = Oracle.scalar_run(dim, n, float(c["tau"]), float(c["kappa"]), float(c["q"]), c["u0"], steps,
                                      src_kind=int(c["src_kind"]), src_params=c["src_params"], family=fam)
        assert rel_gap(c["u"], u) <= 1e-13
    else:
        u, v, nn, tt = Oracle.system_run(dim, n, float(c["tau"]), float(c["ku"]), float(c["kv"]), float(c["q"]),
                                         c["u0"], c["v0"], steps, src_kind=int(c["src_kind"]),
                                         src_params=c["src_params"], family=fam)
        assert rel_gap(c["u"], u) <= 1e-13 and rel_gap(c["v"], v) <= 1e-13
    assert nn == int(c["n_out"]) and tt == pytest.approx(float(c["t_out"]), abs=0)


def test_oracle_setup_matches_reference_golden():
    s = load(os.path.join(GOLD, "setup.npz"))
    for key in [k for k in s if k.startswith("P_")]:
        _, n, dim = key.split("_")
        n, dim = int(n), int(dim)
        dg, of, kappa, q = s[f"diag_off_{n}_{dim}"]
        dg2, of2 = Oracle.operator(dim, n, kappa, q)
        assert dg2 == dg and of2 == of
        P, lam = Oracle.spectral_factor(n, dg, of)
        assert np.array_equal(P, s[key])
        assert np.max(np.abs(lam - s[f"lam_{n}_{dim}"])) <= 1e-15 * np.max(np.abs(lam))
        for fam in (0, 1):
            for ell in (1, 2, 3):
                d = Oracle.dvector(s[f"lam_{n}_{dim}"], 0.01, fam, ell)
                assert rel_gap(s[f"d_{n}_{dim}_{fam}_{ell}"], d) <= 1e-14
    for fam in (0, 1):
        assert np.max(np.abs(Oracle.scheme(fam) - s[f"scheme_{fam}"])) <= 1e-15


def test_oracle_abort_semantics():
    """StepperAbort reports the input state's t and n (test_stepper.cpp:304-321)."""
    from oracle import OracleAbort
    u0 = np.random.default_rng(7).uniform(-0.5, 0.5, 49)
    with pytest.raises(OracleAbort) as ei:
        Oracle.scalar_run(2, 7, 0.01, 1.0, 1.0, u0, 1, src_kind=3, n0=4, t0=0.25)
    assert ei.value.t == 0.25 and ei.value.step == 4


@pytest.mark.skipif(not Ref.available(), reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("dim,n,fam", [(2, 14, 0), (3, 7, 1), (2, 33, 1)])
def test_oracle_matches_live_reference(dim, n, fam):
    u0 = np.random.default_rng(dim * n).uniform(-1, 1, n ** dim)
    a = Ref.scalar_run(dim, n, 0.02, 0.8, 0.5, u0, 3, src_kind=1, family=fam)[0]
    b = Oracle.scalar_run(dim, n, 0.02, 0.8, 0.5, u0, 3, src_kind=1, family=fam)[0]
    assert rel_gap(a, b) <= 1e-13
    v0 = np.random.default_rng(1).uniform(-1, 1, n ** dim)
    a = Ref.system_run(dim, n, 0.05, 1e-3, 5e-4, 0.0, u0, v0, 3, family=fam)
    b = Oracle.system_run(dim, n, 0.05, 1e-3, 5e-4, 0.0, u0, v0, 3, family=fam)
    assert rel_gap(a[0], b[0]) <= 1e-13 and rel_gap(a[1], b[1]) <= 1e-13


@pytest.mark.skipif(not Ref.available(), reason="oracle/_ref not built (needs /root/reference)")
def test_composed_3d_system_reduces_to_reference_scalar_step():
    """The 3D two-species composition (reference has no 3D system stepper) equals
    the reference etd2rkds_step_3d on a decoupled mirrored system."""
    n = 9
    u0 = np.random.default_rng(5).uniform(-1, 1, n ** 3)
    a = Ref.system_run(3, n, 0.01, 0.5, 0.5, 0.0, u0, u0, 4, src_kind=12)
    b = Ref.scalar_run(3, n, 0.01, 0.5, 0.0, u0, 4, src_kind=1)
    assert rel_gap(b[0], a[0]) <= 1e-14 and rel_gap(b[0], a[1]) <= 1e-14


@pytest.mark.parametrize("dim,n", [(2, 13), (3, 7), (2, 24)])
@pytest.mark.parametrize("family", [0, 1])
def test_oracle_thomas_vs_reference(dim, n, family):
    """The C restatement of BackendKind::Thomas (thomas.cpp) against the reference's
    own Thomas path: apply_Q on every axis and ell, scalar and system steps."""
    if not Ref.available():
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(31)
    x = rng.uniform(-1, 1, n ** dim)
    for axis in range(dim):
        for ell in (1, 2, 3):
            a = Ref.apply_q_thomas(dim, n, 0.02, 0.7, 1.0, family, ell, axis, x)
            b = Oracle.apply_q(dim, n, 0.02, 0.7, 1.0, family, ell, axis, x, backend=1)
            assert rel_gap(a, b) <= 1e-14, (axis, ell)
    a = Ref.scalar_run(dim, n, 0.01, 1.0, 1.0, x, 3, src_kind=1, family=family, backend=1)[0]
    th = Oracle.scalar_run(dim, n, 0.01, 1.0, 1.0, x, 3, src_kind=1, family=family, backend=1)[0]
    assert rel_gap(a, th) <= 1e-13
    v = rng.uniform(-1, 1, n ** dim)
    a = Ref.system_run(dim, n, 0.05, 1e-3, 5e-4, 0.0, x, v, 3, family=family, backend=1)
    b = Oracle.system_run(dim, n, 0.05, 1e-3, 5e-4, 0.0, x, v, 3, family=family, backend=1)
    assert rel_gap(a[0], b[0]) <= 1e-13 and rel_gap(a[1], b[1]) <= 1e-13
    # and the two backends of the restatement agree (the reference's backend cross-check)
    sp = Oracle.scalar_run(dim, n, 0.01, 1.0, 1.0, x, 3, src_kind=1, family=family, backend=0)[0]
    assert rel_gap(sp, th) <= 1e-11
