"""TEST INFRASTRUCTURE ONLY — CPU oracle bindings.

Two CPU implementations of the ETD2RK-DS spectral step, used as the checker:

* ``Ref``    — the UNMODIFIED reference library (``/root/reference/proj/core``)
               compiled by ``oracle/Makefile`` into ``oracle/_ref/libetdrd_ref.so``
               together with ``oracle/ref_driver.cpp`` (an extern "C" driver over the
               reference's make_plan/advance/make_system_plan/etd2rkds_step_system).
* ``Oracle`` — the plain-C restatement ``oracle/etd_oracle.c``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU leg may import
this package.  The product (``paper_2601_06849_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(_HERE, "_ref", "libetdrd_ref.so")
ORACLE_SO = os.path.join(_HERE, "_build", "libetd_oracle.so")

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")


class OracleAbort(RuntimeError):
    """Mirror of etdrd::StepperAbort (errors.hpp:22-28)."""

    def __init__(self, msg: str, t: float, step: int):
        super().__init__(msg)
        self.t = t
        self.step = step


def build(quiet: bool = True) -> None:
    """Compile the oracle (and oracle/_ref when /root/reference is present)."""
    out = subprocess.run(["make", "-C", _HERE, "-j8"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


def _check(rc: int, err: bytes, t_ab: float, step_ab: int) -> None:
    if rc == 0:
        return
    msg = err.decode(errors="replace") if err else ""
    if rc == 3:
        raise OracleAbort(msg or "non-finite", t_ab, step_ab)
    if rc == 1:
        raise ValueError(msg or "config error")
    raise RuntimeError(f"oracle rc={rc}: {msg}")


def _params(p) -> np.ndarray:
    a = np.zeros(8)
    if p is not None:
        a[: len(p)] = p
    return a


class Ref:
    """ctypes view of oracle/_ref/libetdrd_ref.so (the reference itself)."""

    _lib = None

    @classmethod
    def lib(cls):
        if cls._lib is None:
            if not os.path.exists(REF_SO):
                raise FileNotFoundError(REF_SO + " (build with `make -C oracle` where /root/reference exists)")
            L = C.CDLL(REF_SO)
            i, d, l = C.c_int, C.c_double, C.c_long
            L.ref_scalar_run.argtypes = [i, i, d, d, d, i, i, i, _dp, _dp, C.POINTER(l), C.POINTER(d), i,
                                         C.POINTER(d), C.c_char_p, i, C.POINTER(d), C.POINTER(l)]
            L.ref_system_run.argtypes = [i, i, d, d, d, d, i, i, i, _dp, _dp, _dp, C.POINTER(l), C.POINTER(d), i, i,
                                         C.POINTER(d), C.c_char_p, i, C.POINTER(d), C.POINTER(l)]
            L.ref_spectral_factor.argtypes = [i, d, d, _dp, _dp]
            L.ref_operator.argtypes = [i, i, i, d, d, C.POINTER(d), C.POINTER(d), C.c_char_p, i]
            L.ref_dvector.argtypes = [i, _dp, d, i, i, _dp]
            L.ref_scheme.argtypes = [i, _dp, C.POINTER(i)]
            L.ref_contract_axis.argtypes = [i, i, i, i, _dp, i, _dp, i, i, _dp, C.c_char_p, i]
            L.ref_apply_q.argtypes = [i, i, d, d, d, i, i, i, _dp, _dp, C.c_char_p, i]
            L.ref_apply_q_thomas.argtypes = [i, i, d, d, d, i, i, i, _dp, _dp, C.c_char_p, i]
            L.ref_sample_step.argtypes = [i, i, i, d, d, d, d, i, i, _dp, C.POINTER(d), C.POINTER(d), _dp,
                                          C.c_char_p, i]
            L.ref_save_field.argtypes = [i, i, i, i, _dp, d, C.c_char_p, C.c_char_p, i]
            L.ref_load_field.argtypes = [C.c_char_p, _dp, C.c_longlong, C.POINTER(C.c_int * 4), C.POINTER(d),
                                         C.c_char_p, i]
            L.ref_set_threads.argtypes = [i]
            L.ref_get_threads.restype = i
            L.ref_blas_config.restype = C.c_char_p
            cls._lib = L
        return cls._lib

    @classmethod
    def available(cls) -> bool:
        return os.path.exists(REF_SO)

    @classmethod
    def set_threads(cls, n: int) -> None:
        cls.lib().ref_set_threads(int(n))

    @classmethod
    def blas_config(cls) -> str:
        return cls.lib().ref_blas_config().decode()

    @classmethod
    def scalar_run(cls, dim, n, tau, kappa, q, u, nsteps, src_kind=1, src_params=None, family=0,
                   backend=0, n0=0, t0=0.0):
        """Returns (u_out, n, t, seconds).  u is x-fastest of length n**dim."""
        u = np.ascontiguousarray(u, dtype=np.float64).copy()
        nn, tt, sec, tab, sab = C.c_long(n0), C.c_double(t0), C.c_double(0), C.c_double(0), C.c_long(0)
        err = C.create_string_buffer(512)
        rc = cls.lib().ref_scalar_run(dim, n, tau, kappa, q, family, backend, src_kind, _params(src_params), u,
                                      C.byref(nn), C.byref(tt), nsteps, C.byref(sec), err, 512,
                                      C.byref(tab), C.byref(sab))
        _check(rc, err.value, tab.value, sab.value)
        return u, nn.value, tt.value, sec.value

    @classmethod
    def system_run(cls, dim, n, tau, ku, kv, q, u, v, nsteps, src_kind=10, src_params=(0.1, 0.01, 0.5),
                   family=0, n0=0, t0=0.0, composed=False, lean=False, inplace=False, backend=0):
        """lean: memory-lean composition (same reference calls, explicit lifetimes);
        inplace: update the given float64 arrays instead of copying them;
        backend: BackendKind (0 Spectral, 1 Thomas)."""
        if not inplace:
            u = np.ascontiguousarray(u, dtype=np.float64).copy()
            v = np.ascontiguousarray(v, dtype=np.float64).copy()
        if lean:
            composed = 2
        nn, tt, sec, tab, sab = C.c_long(n0), C.c_double(t0), C.c_double(0), C.c_double(0), C.c_long(0)
        err = C.create_string_buffer(512)
        rc = cls.lib().ref_system_run(dim, n, tau, ku, kv, q, family, backend, src_kind, _params(src_params), u, v,
                                      C.byref(nn), C.byref(tt), nsteps, int(composed), C.byref(sec), err, 512,
                                      C.byref(tab), C.byref(sab))
        _check(rc, err.value, tab.value, sab.value)
        return u, v, nn.value, tt.value, sec.value

    @classmethod
    def sample_step(cls, n, nsub, nspecies, tau, kappas, q, src_kind, src_params=None, family=0):
        """Bounded reference-step sample at full pencil length n (see ref_driver.cpp).
        Returns (seconds_for_sample_points, sample_points, parts)."""
        sec, pts = C.c_double(), C.c_double()
        parts = np.zeros(3)
        err = C.create_string_buffer(512)
        k1 = kappas[1] if len(kappas) > 1 else 0.0
        rc = cls.lib().ref_sample_step(n, nsub, nspecies, tau, kappas[0], k1, q, family, src_kind,
                                       _params(src_params), C.byref(sec), C.byref(pts), parts, err, 512)
        _check(rc, err.value, 0, 0)
        return sec.value, pts.value, parts

    @classmethod
    def save_field(cls, shape, data, t, path):
        nx, ny, nz = shape
        err = C.create_string_buffer(256)
        rc = cls.lib().ref_save_field(3 if nz > 1 else 2, nx, ny, nz, np.ascontiguousarray(data, dtype=np.float64),
                                      t, path.encode(), err, 256)
        _check(rc, err.value, 0, 0)

    @classmethod
    def load_field(cls, path, cap):
        out = np.zeros(cap)
        shape = (C.c_int * 4)()
        t = C.c_double()
        err = C.create_string_buffer(256)
        rc = cls.lib().ref_load_field(path.encode(), out, cap, C.byref(shape), C.byref(t), err, 256)
        _check(rc, err.value, 0, 0)
        n = shape[1] * shape[2] * shape[3]
        return out[:n], tuple(shape), t.value

    @classmethod
    def operator(cls, dim, n, axis, kappa, q):
        dg, of = C.c_double(), C.c_double()
        err = C.create_string_buffer(256)
        rc = cls.lib().ref_operator(dim, n, axis, kappa, q, C.byref(dg), C.byref(of), err, 256)
        _check(rc, err.value, 0, 0)
        return dg.value, of.value

    @classmethod
    def spectral_factor(cls, n, diag, off):
        P = np.zeros(n * n)
        e = np.zeros(n)
        cls.lib().ref_spectral_factor(n, diag, off, P, e)
        return P, e

    @classmethod
    def dvector(cls, eig, tau, family, ell):
        eig = np.ascontiguousarray(eig, dtype=np.float64)
        d = np.zeros(len(eig))
        cls.lib().ref_dvector(len(eig), eig, tau, family, ell, d)
        return d

    @classmethod
    def scheme(cls, family):
        out = np.zeros(3 * 2 * 4)
        nt = C.c_int()
        cls.lib().ref_scheme(family, out, C.byref(nt))
        return out[: 3 * nt.value * 4].reshape(3, nt.value, 4)

    @classmethod
    def contract_axis(cls, shape, M, n, x, axis, transpose):
        nx, ny, nz = shape
        dim = 3 if nz > 1 else 2
        out = np.zeros(nx * ny * nz)
        err = C.create_string_buffer(256)
        rc = cls.lib().ref_contract_axis(dim, nx, ny, nz, np.ascontiguousarray(M, dtype=np.float64), n,
                                         np.ascontiguousarray(x, dtype=np.float64), axis, int(transpose), out,
                                         err, 256)
        _check(rc, err.value, 0, 0)
        return out

    @classmethod
    def apply_q(cls, dim, n, tau, kappa, q, family, ell, axis, x):
        out = np.zeros(n ** dim)
        err = C.create_string_buffer(256)
        rc = cls.lib().ref_apply_q(dim, n, tau, kappa, q, family, ell, axis,
                                   np.ascontiguousarray(x, dtype=np.float64), out, err, 256)
        _check(rc, err.value, 0, 0)
        return out

    @classmethod
    def apply_q_thomas(cls, dim, n, tau, kappa, q, family, ell, axis, x):
        """apply_Q_thomas (thomas.cpp:128-160)."""
        out = np.zeros(n ** dim)
        err = C.create_string_buffer(256)
        rc = cls.lib().ref_apply_q_thomas(dim, n, tau, kappa, q, family, ell, axis,
                                          np.ascontiguousarray(x, dtype=np.float64), out, err, 256)
        _check(rc, err.value, 0, 0)
        return out


class Oracle:
    """ctypes view of oracle/_build/libetd_oracle.so (the plain-C restatement)."""

    _lib = None

    @classmethod
    def lib(cls):
        if cls._lib is None:
            if not os.path.exists(ORACLE_SO):
                build()
            L = C.CDLL(ORACLE_SO)
            i, d, l = C.c_int, C.c_double, C.c_long
            L.etd_o_operator.argtypes = [i, i, d, d, C.POINTER(d), C.POINTER(d)]
            L.etd_o_spectral_factor.argtypes = [i, d, d, _dp, _dp]
            L.etd_o_scheme.argtypes = [i, _dp, C.POINTER(i)]
            L.etd_o_dvector.argtypes = [i, _dp, d, i, i, _dp]
            L.etd_o_contract.argtypes = [i, i, i, _dp, i, i, _dp, _dp]
            L.etd_o_apply_q.argtypes = [i, i, d, d, d, i, i, i, _dp, _dp]
            L.etd_o_scalar_run.argtypes = [i, i, d, d, d, i, i, _dp, _dp, C.POINTER(l), C.POINTER(d), i,
                                           C.POINTER(d), C.POINTER(l)]
            L.etd_o_system_run.argtypes = [i, i, d, d, d, d, i, i, _dp, _dp, _dp, C.POINTER(l), C.POINTER(d), i,
                                           C.POINTER(d), C.POINTER(l)]
            L.etd_o_apply_q_b.argtypes = [i, i, d, d, d, i, i, i, i, _dp, _dp]
            L.etd_o_scalar_run_b.argtypes = [i, i, d, d, d, i, i, i, _dp, _dp, C.POINTER(l), C.POINTER(d), i,
                                             C.POINTER(d), C.POINTER(l)]
            L.etd_o_system_run_b.argtypes = [i, i, d, d, d, d, i, i, i, _dp, _dp, _dp, C.POINTER(l), C.POINTER(d),
                                             i, C.POINTER(d), C.POINTER(l)]
            cls._lib = L
        return cls._lib

    @classmethod
    def operator(cls, dim, n, kappa, q):
        dg, of = C.c_double(), C.c_double()
        cls.lib().etd_o_operator(dim, n, kappa, q, C.byref(dg), C.byref(of))
        return dg.value, of.value

    @classmethod
    def spectral_factor(cls, n, diag, off):
        P = np.zeros(n * n)
        e = np.zeros(n)
        cls.lib().etd_o_spectral_factor(n, diag, off, P, e)
        return P, e

    @classmethod
    def scheme(cls, family):
        out = np.zeros(3 * 2 * 4)
        nt = C.c_int()
        rc = cls.lib().etd_o_scheme(family, out, C.byref(nt))
        if rc:
            raise RuntimeError("scheme construction failed")
        return out[: 3 * nt.value * 4].reshape(3, nt.value, 4)

    @classmethod
    def dvector(cls, eig, tau, family, ell):
        eig = np.ascontiguousarray(eig, dtype=np.float64)
        d = np.zeros(len(eig))
        cls.lib().etd_o_dvector(len(eig), eig, tau, family, ell, d)
        return d

    @classmethod
    def contract(cls, shape, M, x, axis, transpose):
        nx, ny, nz = shape
        out = np.zeros(nx * ny * nz)
        cls.lib().etd_o_contract(nx, ny, nz, np.ascontiguousarray(M, dtype=np.float64), axis, int(transpose),
                                 np.ascontiguousarray(x, dtype=np.float64), out)
        return out

    @classmethod
    def apply_q(cls, dim, n, tau, kappa, q, family, ell, axis, x, backend=0):
        """backend 0: spectral (tensor_ops.cpp:164-172); 1: Thomas (thomas.cpp:128-160)."""
        out = np.zeros(n ** dim)
        cls.lib().etd_o_apply_q_b(dim, n, tau, kappa, q, family, backend, ell, axis,
                                  np.ascontiguousarray(x, dtype=np.float64), out)
        return out

    @classmethod
    def scalar_run(cls, dim, n, tau, kappa, q, u, nsteps, src_kind=1, src_params=None, family=0, n0=0, t0=0.0,
                   backend=0):
        u = np.ascontiguousarray(u, dtype=np.float64).copy()
        nn, tt, tab, sab = C.c_long(n0), C.c_double(t0), C.c_double(0), C.c_long(0)
        rc = cls.lib().etd_o_scalar_run_b(dim, n, tau, kappa, q, family, backend, src_kind, _params(src_params), u,
                                          C.byref(nn), C.byref(tt), nsteps, C.byref(tab), C.byref(sab))
        _check(rc, b"", tab.value, sab.value)
        return u, nn.value, tt.value

    @classmethod
    def system_run(cls, dim, n, tau, ku, kv, q, u, v, nsteps, src_kind=10, src_params=(0.1, 0.01, 0.5),
                   family=0, n0=0, t0=0.0, backend=0):
        u = np.ascontiguousarray(u, dtype=np.float64).copy()
        v = np.ascontiguousarray(v, dtype=np.float64).copy()
        nn, tt, tab, sab = C.c_long(n0), C.c_double(t0), C.c_double(0), C.c_long(0)
        rc = cls.lib().etd_o_system_run_b(dim, n, tau, ku, kv, q, family, backend, src_kind, _params(src_params),
                                          u, v, C.byref(nn), C.byref(tt), nsteps, C.byref(tab), C.byref(sab))
        _check(rc, b"", tab.value, sab.value)
        return u, v, nn.value, tt.value


def rel_gap(a, b) -> float:
    """max|a-b| / max|a| — the reference's normwise metric (test_stepper.cpp:50-57)."""
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    den = max(float(np.max(np.abs(a))) if a.size else 0.0, 1e-300)
    return float(np.max(np.abs(a - b))) / den if a.size else 0.0
