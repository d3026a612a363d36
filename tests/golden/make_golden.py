"""Generate tests/golden/*.npz from the REFERENCE ITSELF (oracle/_ref/libetdrd_ref.so,
the unmodified etdrd core compiled from /root/reference/proj/core/src).

Run in the build container (needs oracle/_ref):  python tests/golden/make_golden.py
The fixtures pin the oracle restatement (tests/test_oracle.py, CPU) and the CUDA
path (tests/test_gpu_golden.py, GPU) to the reference's own outputs.
"""
import os
import sys

import zlib

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import Ref  # noqa: E402

Ref.set_threads(1)  # deterministic BLAS summation order for the fixtures


def rng_field(seed, n):
    return np.random.default_rng(seed).uniform(-1.0, 1.0, n)


def main():
    cases = {}
    # ---- scalar steps (make_plan + advance; stepper.cpp:182-257) ----
    scalar = [
        ("scalar2d_p02", 2, 15, 0.01, 1.0, 1.0, 0, 1, None, 5),
        ("scalar2d_p04", 2, 12, 0.02, 1.3, 0.7, 1, 1, None, 4),
        ("scalar3d_p02", 3, 9, 0.01, 0.5, 1.0, 0, 1, None, 4),
        ("scalar3d_p04", 3, 8, 0.02, 1.0, 0.0, 1, 1, None, 3),
        ("scalar2d_poly", 2, 10, 0.01, 1.0, 1.0, 0, 2, (0.05, -0.3, 0.2, -1.0), 6),
        ("cfg0_physics_n31", 2, 31, 1e-3, 1.0, 1.0, 0, 1, None, 10),
        ("cfg2_physics_n15", 3, 15, 1e-3, 0.1, 1.0, 0, 1, None, 5),
        # catalogue sources (problems.cpp): manufactured Allen-Cahn (p0 lambda, p1 lin, p2 kappa), singular
        ("ac_manufactured2d_p02", 2, 20, 0.02, 1.0, 0.0, 0, 4, (1.0, -1.0 + 2 * np.pi ** 2, 1.0), 5),
        ("ac_manufactured3d_p04", 3, 10, 0.02, 1.0, 0.0, 1, 4, (1.0, -1.0 + 3 * np.pi ** 2, 1.0), 4),
        ("singular2d_p02", 2, 16, 0.01, 1.0, 1.0, 0, 5, (0.1,), 5),
    ]
    for name, dim, n, tau, kappa, q, fam, kind, params, steps in scalar:
        u0 = rng_field(zlib.crc32(name.encode()), n ** dim)
        if kind in (4, 5):
            u0 = 0.4 * (u0 + 1.0)  # inside the singular source's domain (u < 1)
        u1, nn, tt, _ = Ref.scalar_run(dim, n, tau, kappa, q, u0, steps, src_kind=kind, src_params=params,
                                       family=fam)
        cases[name] = dict(kind="scalar", dim=dim, n=n, tau=tau, kappa=kappa, q=q, family=fam, src_kind=kind,
                           src_params=np.array(params or (0.0,) * 4, dtype=float), steps=steps, u0=u0, u=u1,
                           n_out=nn, t_out=tt)
    # ---- two-species steps (system_stepper.cpp:74-114; 3D composed) ----
    system = [
        ("system2d_fhn", 2, 15, 0.05, 1e-3, 5e-4, 0.0, 0, 10, (0.1, 0.01, 0.5), 5),
        ("system2d_fhn_classic_p04", 2, 12, 0.01, 0.01, 10.0, 0.0, 1, 11, (1.0, 1.0), 4),
        ("system3d_fhn", 3, 9, 0.05, 1e-3, 5e-4, 0.0, 0, 10, (0.1, 0.01, 0.5), 4),
        # q != 0: the unit-kappa operator carries q/dim per axis and kappa_c scales the
        # whole eigenvalue, q term included (system_stepper.cpp:52-61)
        ("system2d_fhn_q", 2, 14, 0.05, 2e-2, 5e-3, 0.6, 1, 10, (0.1, 0.01, 0.5), 4),
        ("system3d_fhn_q", 3, 10, 0.05, 2e-2, 5e-3, 0.9, 0, 10, (0.1, 0.01, 0.5), 3),
        ("cfg4_physics_n11", 3, 11, 0.05, 1e-3, 5e-4, 0.0, 0, 10, (0.1, 0.01, 0.5), 3),
    ]
    for name, dim, n, tau, ku, kv, q, fam, kind, params, steps in system:
        s = zlib.crc32(name.encode())
        u0, v0 = rng_field(s, n ** dim), 0.5 * rng_field(s + 1, n ** dim)
        u1, v1, nn, tt, _ = Ref.system_run(dim, n, tau, ku, kv, q, u0, v0, steps, src_kind=kind,
                                           src_params=params, family=fam)
        cases[name] = dict(kind="system", dim=dim, n=n, tau=tau, ku=ku, kv=kv, q=q, family=fam, src_kind=kind,
                           src_params=np.array(params, dtype=float), steps=steps, u0=u0, v0=v0, u=u1, v=v1,
                           n_out=nn, t_out=tt)
    for name, c in cases.items():
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **c)
    # ---- host setup (operators.cpp:11-56, rational.cpp:133-198) ----
    setup = {}
    for n, dim, kappa, q in ((15, 2, 1.0, 1.0), (31, 3, 0.1, 1.0), (64, 2, 0.5, 0.0)):
        dg, of = Ref.operator(dim, n, 0, kappa, q)
        P, lam = Ref.spectral_factor(n, dg, of)
        setup[f"P_{n}_{dim}"] = P
        setup[f"lam_{n}_{dim}"] = lam
        setup[f"diag_off_{n}_{dim}"] = np.array([dg, of, kappa, q])
        for fam in (0, 1):
            for ell in (1, 2, 3):
                setup[f"d_{n}_{dim}_{fam}_{ell}"] = Ref.dvector(lam, 0.01, fam, ell)
    for fam in (0, 1):
        setup[f"scheme_{fam}"] = Ref.scheme(fam)
    np.savez_compressed(os.path.join(HERE, "setup.npz"), **setup)
    print(f"wrote {len(cases)} step fixtures + setup.npz")


if __name__ == "__main__":
    main()
