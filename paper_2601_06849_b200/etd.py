"""Host-side mirror of the reference stepper API over the C-ABI (include/etd_b200.h).

The reference (`etdrd`, C++) exposes the ETD2RK-DS spectral step as

    Grid unit_box_grid(dim, m);                                   grid.hpp:43-47
    StepperPlan make_plan(grid, tau, kappa, q, scheme, backend);  stepper.hpp:59-61
    StepperState advance(plan, state, f);                         stepper.hpp:85-86
    SystemPlan make_system_plan(grid, tau, ku, kv, q, scheme, backend);   stepper.hpp:107-108
    SystemState etd2rkds_step_system(plan, state, f);             stepper.hpp:116-117

with exceptions ConfigError / NumericsError / StepperAbort{t, step} /
MemoryGuardError (errors.hpp:8-30).  This module keeps those names, argument
meanings and error behaviour; the work runs in ``libetd_b200.so`` (sm_100a).
There is no CPU fallback: without the extension or without a B200 every call
that would compute raises.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libetd_b200.so")


# ----------------------------------------------------------------- errors (errors.hpp)
class ConfigError(ValueError):
    """etdrd::ConfigError — bad input / malformed configuration (CLI exit 2)."""


class NumericsError(RuntimeError):
    """etdrd::NumericsError."""


class StepperAbort(RuntimeError):
    """etdrd::StepperAbort — non-finite value; t and step of the INPUT state."""

    def __init__(self, msg: str, t: float, step: int):
        super().__init__(msg)
        self.t = t
        self.step = step


class MemoryGuardError(RuntimeError):
    """etdrd::MemoryGuardError."""


class DeviceError(RuntimeError):
    """CUDA failure or no usable B200 (no reference equivalent; no CPU fallback)."""


ETD_OK, ETD_ERR_CONFIG, ETD_ERR_NUMERICS, ETD_ERR_ABORT, ETD_ERR_MEMORY, ETD_ERR_CUDA, ETD_ERR_NODEVICE = range(7)


class PadeFamily(enum.IntEnum):
    """rational.hpp:31"""
    P02 = 0
    P04 = 1


EXACT_FAMILY = 2  # etd_family ETD_EXACT


class BackendKind(enum.IntEnum):
    """tensor_ops.hpp:31 plus the B200 backends this package adds.  Spectral and
    Thomas select the device implementations of the same backends (CudaSpectral,
    CudaThomas); NonSplitBanded is not implemented (out of scope)."""
    Spectral = 0
    Thomas = 1
    NonSplitBanded = 2
    ExactExpReference = 3
    CudaSpectral = 100
    CudaThomas = 101


_DEVICE_BACKEND = {BackendKind.Spectral: 0, BackendKind.CudaSpectral: 0,
                   BackendKind.Thomas: 1, BackendKind.CudaThomas: 1}


class SourceKind(enum.IntEnum):
    """include/etd_b200.h etd_source_kind"""
    ZERO = 0
    AC_CUBIC = 1
    POLY3 = 2
    NAN_PROBE = 3
    AC_MANUFACTURED = 4
    SINGULAR = 5
    FHN_CUBIC = 10
    FHN_CLASSIC = 11
    MIRROR_AC = 12
    DECOUPLED = 13


@dataclass(frozen=True)
class DeviceSource:
    """Device stand-in for the reference SourceFunction/SystemSource (stepper.hpp:18-29).

    A std::function cannot run on the GPU, so the CUDA backend takes a pointwise
    kind + parameters.  Passing anything else raises ConfigError (no CPU fallback).
    """
    kind: SourceKind
    params: tuple = ()
    autonomous: bool = True

    def params8(self):
        p = list(self.params)[:8]
        return p + [0.0] * (8 - len(p))


def allen_cahn_cubic() -> DeviceSource:
    """f(u) = u - u^3 (BASELINE configs 0-2)."""
    return DeviceSource(SourceKind.AC_CUBIC)


def fhn_cubic(a: float = 0.1, eps: float = 0.01, beta: float = 0.5) -> DeviceSource:
    """fu = u(1-u)(u-a) - v ; fv = eps(beta u - v) (BASELINE configs 3-4)."""
    return DeviceSource(SourceKind.FHN_CUBIC, (a, eps, beta))


def fhn_classic(eps: float = 1.0, alpha: float = 1.0) -> DeviceSource:
    """fu = u - u^3/3 - v ; fv = eps(u - alpha v) (reference problems.cpp:170-171)."""
    return DeviceSource(SourceKind.FHN_CLASSIC, (eps, alpha))


def allen_cahn_manufactured(dim: int, lam: float = 1.0, kappa: float = 1.0) -> DeviceSource:
    """Catalogue Allen-Cahn source with the manufactured forcing that pins the
    decaying sine-product solution u* = e^{-lam t} prod sin(pi x_a)
    (reference problems.cpp:68-106; non-autonomous)."""
    import math
    lin = -lam + kappa * dim * math.pi * math.pi  # problems.cpp:91
    return DeviceSource(SourceKind.AC_MANUFACTURED, (lam, lin, kappa, float(dim)), autonomous=False)


def singular(rho: float = 0.1) -> DeviceSource:
    """rho u/(1-u) with the domain guard u >= 1 -> StepperAbort(t, -1) (problems.cpp:108-136)."""
    return DeviceSource(SourceKind.SINGULAR, (rho,))


def poly3(p0=0.0, p1=0.0, p2=0.0, p3=0.0) -> DeviceSource:
    return DeviceSource(SourceKind.POLY3, (p0, p1, p2, p3))


# ----------------------------------------------------------------- grid (grid.hpp)
@dataclass
class Grid:
    """Uniform tensor grid; m[a] counts SUBINTERVALS, interior = m[a]-1 (grid.hpp:14-16)."""
    dim: int = 2
    low: tuple = (0.0, 0.0, 0.0)
    high: tuple = (1.0, 1.0, 1.0)
    m: tuple = (2, 2, 1)

    @property
    def h(self):
        return tuple((self.high[a] - self.low[a]) / self.m[a] for a in range(3))

    def interior(self, a: int) -> int:
        return self.m[a] - 1

    def interior_shape(self):
        """(nx, ny, nz) with nz = 1 in 2D (grid.hpp:31-33)."""
        return (self.m[0] - 1, self.m[1] - 1, self.m[2] - 1 if self.dim == 3 else 1)

    def total_interior(self) -> int:
        nx, ny, nz = self.interior_shape()
        return nx * ny * nz

    def coord(self, a: int, i: int) -> float:
        return self.low[a] + (i + 1) * self.h[a]


def build_grid(dim: int, bounds: Sequence[tuple], m_per_axis: Sequence[int]) -> Grid:
    """grid.cpp:9-34 validation semantics."""
    if dim not in (2, 3):
        raise ConfigError(f"grid dimension must be 2 or 3, got {dim}")
    if len(bounds) != dim or len(m_per_axis) != dim:
        raise ConfigError("bounds/m arrays must have one entry per dimension")
    low, high, m = [0.0] * 3, [1.0] * 3, [1, 1, 1]
    for a in range(dim):
        lo, hi = bounds[a]
        if not hi > lo:
            raise ConfigError(f"axis {a}: upper bound must exceed lower")
        if m_per_axis[a] < 2:
            raise ConfigError(f"axis {a}: need at least 2 subintervals for a nonempty interior")
        low[a], high[a], m[a] = float(lo), float(hi), int(m_per_axis[a])
    return Grid(dim, tuple(low), tuple(high), tuple(m))


def unit_box_grid(dim: int, m: int) -> Grid:
    """grid.cpp:36-42"""
    return build_grid(dim, [(0.0, 1.0)] * dim, [m] * dim)


# ----------------------------------------------------------------- ctypes binding
class _Desc(C.Structure):
    _fields_ = [
        ("dim", C.c_int), ("n", C.c_int * 3), ("low", C.c_double * 3), ("high", C.c_double * 3),
        ("tau", C.c_double), ("family", C.c_int), ("nspecies", C.c_int), ("kappa", C.c_double * 2),
        ("q", C.c_double), ("src_kind", C.c_int), ("src_params", C.c_double * 8), ("device", C.c_int),
        ("world_size", C.c_int), ("rank", C.c_int), ("nccl_unique_id", C.c_void_p), ("backend", C.c_int),
        ("memory_cap_bytes", C.c_ulonglong),
    ]


_lib = None
_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")


def lib():
    """Load libetd_b200.so (built in-tree).  Fails loudly when it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise DeviceError(f"{LIB_PATH} missing: build it with `python -m paper_2601_06849_b200.build`")
        L = C.CDLL(LIB_PATH)
        i, d, l, vp, sz = C.c_int, C.c_double, C.c_long, C.c_void_p, C.c_size_t
        L.etd_create.argtypes = [C.POINTER(_Desc), C.POINTER(vp)]
        L.etd_destroy.argtypes = [vp]
        L.etd_plan_device_bytes.argtypes = [C.POINTER(_Desc), C.POINTER(C.c_ulonglong)]
        L.etd_slab_range.argtypes = [vp, C.POINTER(i), C.POINTER(i)]
        L.etd_set_state.argtypes = [vp, i, vp, sz, l, d]
        L.etd_get_state.argtypes = [vp, i, vp, sz, C.POINTER(l), C.POINTER(d)]
        L.etd_step.argtypes = [vp, i]
        L.etd_advance.argtypes = [vp, vp, vp, l, d, i, vp, vp, C.POINTER(l), C.POINTER(d)]
        L.etd_set_source.argtypes = [vp, i, vp]
        L.etd_last_error.argtypes = [vp, C.c_char_p, sz, C.POINTER(d), C.POINTER(l)]
        L.etd_stream.argtypes = [vp]
        L.etd_stream.restype = C.c_ulonglong
        L.etd_launches_per_step.argtypes = [vp]
        L.etd_comm_ranks.argtypes = [vp, C.POINTER(i)]
        L.etd_set_profiling.argtypes = [vp, i]
        L.etd_stage_count.argtypes = [vp]
        L.etd_stage_info.argtypes = [vp, i, C.c_char_p, sz, C.POINTER(d), C.POINTER(l), C.POINTER(d), C.POINTER(d)]
        L.etd_stage_flops.argtypes = [vp, i, C.POINTER(d), C.POINTER(d)]
        L.etd_parity_split.argtypes = [vp, C.POINTER(C.c_int)]
        L.etd_setup_fold_matrices.argtypes = [i, i, vp, vp]
        L.etd_setup_fold2_matrices.argtypes = [i, i, vp, vp, vp, vp, vp]
        L.etd_setup_back6_matrix.argtypes = [i, i, vp]
        L.etd_fold_level.argtypes = [vp, C.POINTER(C.c_int)]
        L.etd_debug_transform.argtypes = [vp, i, i, i, i, i, vp, vp]
        L.etd_fill_config_ic.argtypes = [i, C.c_ulonglong, i, i, i, i, vp]
        L.etd_setup_axis.argtypes = [i, d, d, i, d, d, vp, vp]
        L.etd_setup_dvector.argtypes = [i, vp, d, i, i, vp]
        L.etd_setup_scheme.argtypes = [i, vp, C.POINTER(i)]
        L.etd_save_snapshot.argtypes = [vp, i, C.c_char_p]
        L.etd_load_snapshot.argtypes = [vp, i, C.c_char_p, l]
        L.etd_zslab_partition.argtypes = [i, i, i, C.POINTER(i), C.POINTER(i)]
        L.etd_nccl_unique_id.argtypes = [vp]
        L.etd_group_step.argtypes = [C.POINTER(vp), i, i]
        L.etd_setup_phi.argtypes = [i, d]
        L.etd_setup_phi.restype = d
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _raise(rc: int, handle) -> None:
    if rc == ETD_OK:
        return
    msg = C.create_string_buffer(1024)
    t, s = C.c_double(), C.c_long()
    lib().etd_last_error(handle, msg, 1024, C.byref(t), C.byref(s))
    text = msg.value.decode(errors="replace")
    if rc == ETD_ERR_ABORT:
        raise StepperAbort(text, t.value, s.value)
    if rc == ETD_ERR_CONFIG:
        raise ConfigError(text)
    if rc == ETD_ERR_NUMERICS:
        raise NumericsError(text)
    if rc == ETD_ERR_MEMORY:
        raise MemoryGuardError(text)
    raise DeviceError(text or f"etd error {rc}")


# ----------------------------------------------------------------- plans
class _Handle:
    def __init__(self, desc: _Desc):
        h = C.c_void_p()
        rc = lib().etd_create(C.byref(desc), C.byref(h))
        _raise(rc, None)
        self.h = h
        self.desc = desc

    def close(self):
        if getattr(self, "h", None):
            lib().etd_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _make_desc(grid: Grid, tau, family, nspecies, kappas, q, source: DeviceSource, device=0,
               world_size=1, rank=0, nccl_id=None, backend=0, memory_cap_bytes=0) -> _Desc:
    d = _Desc()
    d.dim = grid.dim
    sh = grid.interior_shape()
    for a in range(3):
        d.n[a] = sh[a] if a < grid.dim else 1
        d.low[a] = grid.low[a]
        d.high[a] = grid.high[a]
    d.tau = float(tau)
    d.family = int(family)
    d.nspecies = nspecies
    d.kappa[0] = float(kappas[0])
    d.kappa[1] = float(kappas[1] if len(kappas) > 1 else 0.0)
    d.q = float(q)
    d.src_kind = int(source.kind)
    for i, v in enumerate(source.params8()):
        d.src_params[i] = float(v)
    d.device = device
    d.world_size = world_size
    d.rank = rank
    d.backend = int(backend)
    d.memory_cap_bytes = int(memory_cap_bytes)
    d.nccl_unique_id = None
    if nccl_id is not None:
        d._id_buf = C.create_string_buffer(bytes(nccl_id), 128)  # kept alive with the desc
        d.nccl_unique_id = C.cast(d._id_buf, C.c_void_p)
    return d


def _family(scheme) -> int:
    if isinstance(scheme, (int, PadeFamily)):
        return int(scheme)
    if isinstance(scheme, str) and scheme.lower() == "exact":
        return EXACT_FAMILY
    if isinstance(scheme, str):
        return {"p02": 0, "p04": 1}[scheme.lower()]
    raise ConfigError("scheme must be a PadeFamily")


def _check_source(src, nspecies):
    if not isinstance(src, DeviceSource):
        raise ConfigError("the CudaSpectral backend needs a DeviceSource descriptor; "
                          "host callables cannot run on the device (no CPU fallback)")
    return src


class _PlanBase:
    nspecies = 1

    def __init__(self, grid: Grid, tau: float, family, kappas, q, source: Optional[DeviceSource], device=0,
                 world_size=1, rank=0, nccl_id=None, backend=BackendKind.CudaSpectral, memory_cap_bytes=0):
        if not tau > 0.0:
            raise ConfigError("tau must be positive")
        self.grid = grid
        self.tau = float(tau)
        fam = _family(family)
        self.family = PadeFamily(fam) if fam in (0, 1) else fam
        self.q = float(q)
        if backend not in _DEVICE_BACKEND:
            raise ConfigError(f"backend {BackendKind(backend).name} is not implemented on the device")
        self.backend = BackendKind.CudaThomas if _DEVICE_BACKEND[backend] == 1 else BackendKind.CudaSpectral
        self._source = source or (allen_cahn_cubic() if self.nspecies == 1 else fhn_cubic())
        self._h = _Handle(_make_desc(grid, tau, self.family, self.nspecies, kappas, q, self._source, device,
                                     world_size, rank, nccl_id, _DEVICE_BACKEND[backend], memory_cap_bytes))
        z0, z1 = C.c_int(), C.c_int()
        lib().etd_slab_range(self._h.h, C.byref(z0), C.byref(z1))
        self.slab = (z0.value, z1.value)
        nx, ny, nz = grid.interior_shape()
        self.local_shape = (nx, ny, z1.value - z0.value if grid.dim == 3 else 1)
        self.local_count = self.local_shape[0] * self.local_shape[1] * self.local_shape[2]

    # -- device-resident interface (extension of the reference API) --
    @property
    def handle(self):
        return self._h.h

    def set_source(self, src: DeviceSource):
        src = _check_source(src, self.nspecies)
        if src != self._source:
            p = np.asarray(src.params8(), dtype=np.float64)
            _raise(lib().etd_set_source(self.handle, int(src.kind), _ptr(p)), self.handle)
            self._source = src

    def upload(self, species: int, values: np.ndarray, n: int = 0, t: float = 0.0):
        a = np.ascontiguousarray(values, dtype=np.float64).reshape(-1)
        if a.size != self.local_count:
            raise ConfigError("state shape does not match plan grid")
        _raise(lib().etd_set_state(self.handle, species, _ptr(a), a.size, int(n), float(t)), self.handle)

    def upload_ptr(self, species: int, host_ptr: int, count: int, n: int = 0, t: float = 0.0):
        """Upload from a raw host pointer (e.g. pinned memory)."""
        _raise(lib().etd_set_state(self.handle, species, C.c_void_p(host_ptr), count, int(n), float(t)),
               self.handle)

    def download(self, species: int = 0, out: Optional[np.ndarray] = None):
        a = np.empty(self.local_count) if out is None else out
        n, t = C.c_long(), C.c_double()
        _raise(lib().etd_get_state(self.handle, species, _ptr(a), a.size, C.byref(n), C.byref(t)), self.handle)
        return a, n.value, t.value

    def download_ptr(self, species: int, host_ptr: int, count: int):
        n, t = C.c_long(), C.c_double()
        _raise(lib().etd_get_state(self.handle, species, C.c_void_p(host_ptr), count, C.byref(n), C.byref(t)),
               self.handle)
        return n.value, t.value

    def advance_ptr(self, u_in: int, v_in: int, u_out: int, v_out: int, n: int = 0, t: float = 0.0,
                    nsteps: int = 1):
        """etd_advance on raw host pointers (pinned buffers overlap the copies with
        compute): upload, nsteps steps, download.  Returns (n, t)."""
        no, to = C.c_long(), C.c_double()
        rc = lib().etd_advance(self.handle, C.c_void_p(u_in), C.c_void_p(v_in or None), int(n), float(t),
                               int(nsteps), C.c_void_p(u_out), C.c_void_p(v_out or None), C.byref(no), C.byref(to))
        _raise(rc, self.handle)
        return no.value, to.value

    def save_snapshot(self, species: int, path: str):
        """ETRD snapshot of the device state (reference save_field, field.cpp:46-58)."""
        _raise(lib().etd_save_snapshot(self.handle, species, os.fsencode(path)), self.handle)

    def load_snapshot(self, species: int, path: str, n: int = -1):
        """Restore a species from an ETRD snapshot (reference load_field, field.cpp:60-81)."""
        _raise(lib().etd_load_snapshot(self.handle, species, os.fsencode(path), int(n)), self.handle)

    def step(self, nsteps: int = 1):
        """Advance the device-resident state nsteps times (StepperAbort on non-finite)."""
        _raise(lib().etd_step(self.handle, int(nsteps)), self.handle)

    @property
    def stream(self) -> int:
        return int(lib().etd_stream(self.handle))

    @property
    def launches_per_step(self) -> int:
        return int(lib().etd_launches_per_step(self.handle))

    def comm_ranks(self) -> int:
        """Ranks of the exchange group (ncclCommCount of an NCCL-sharded plan)."""
        out = C.c_int()
        _raise(lib().etd_comm_ranks(self.handle, C.byref(out)), self.handle)
        return out.value

    def set_profiling(self, on: bool):
        lib().etd_set_profiling(self.handle, int(bool(on)))

    def stage_stats(self):
        out = []
        for i in range(lib().etd_stage_count(self.handle)):
            name = C.create_string_buffer(64)
            ms, la, fl, by = C.c_double(), C.c_long(), C.c_double(), C.c_double()
            lib().etd_stage_info(self.handle, i, name, 64, C.byref(ms), C.byref(la), C.byref(fl), C.byref(by))
            ex, dn = C.c_double(), C.c_double()
            lib().etd_stage_flops(self.handle, i, C.byref(ex), C.byref(dn))
            out.append({"name": name.value.decode(), "ms_total": ms.value, "launches": la.value,
                        "flops_per_launch": fl.value, "bytes_per_launch": by.value,
                        "dense_flops_per_launch": dn.value})
        return out

    def parity_split(self) -> tuple:
        """Per axis: whether the eigenbasis transforms run parity-split (h x h halves)."""
        a = (C.c_int * 3)()
        _raise(lib().etd_parity_split(self.handle, a), self.handle)
        return tuple(bool(a[i]) for i in range(self.grid.dim))

    def fold_level(self) -> tuple:
        """Per axis: 0 dense, 1 first-level parity split, 2 second level (§4b)."""
        a = (C.c_int * 3)()
        _raise(lib().etd_fold_level(self.handle, a), self.handle)
        return tuple(a[i] for i in range(self.grid.dim))

    def debug_transform(self, x: np.ndarray, axis: int, back: bool = False, ell: int = 0, apply_q: bool = False,
                        species: int = 0) -> np.ndarray:
        a = np.ascontiguousarray(x, dtype=np.float64).reshape(-1)
        out = np.empty_like(a)
        _raise(lib().etd_debug_transform(self.handle, species, axis, int(back), ell, int(apply_q), _ptr(a),
                                         _ptr(out)), self.handle)
        return out

    def apply_Q(self, ell: int, field_values: np.ndarray, axis: int, species: int = 0) -> np.ndarray:
        """StepperPlan::apply_Q (stepper.cpp:106-116): Q_ell(tau A_axis) applied along
        `axis` to a host field, on the plan's backend (eigenbasis transforms or Thomas)."""
        if ell < 1 or ell > 3:
            raise ConfigError("ell must be 1, 2, or 3")
        return self.debug_transform(field_values, axis, ell=ell, apply_q=True, species=species)

    def close(self):
        self._h.close()


class StepperPlan(_PlanBase):
    """make_plan(...) result for BackendKind.CudaSpectral (stepper.hpp:35-56)."""
    nspecies = 1

    def __init__(self, grid, tau, kappa, q, family=PadeFamily.P02, source=None, device=0, world_size=1, rank=0,
                 nccl_id=None, backend=BackendKind.CudaSpectral, memory_cap_bytes=0):
        if not kappa > 0.0:
            raise ConfigError("diffusivity must be positive")
        self.kappa = float(kappa)
        super().__init__(grid, tau, family, (kappa,), q, source, device, world_size, rank, nccl_id, backend,
                         memory_cap_bytes)


class SystemPlan(_PlanBase):
    """make_system_plan(...) for BackendKind.CudaSpectral, 2D and 3D (stepper.hpp:91-108)."""
    nspecies = 2

    def __init__(self, grid, tau, kappa_u, kappa_v, q, family=PadeFamily.P02, source=None, device=0,
                 world_size=1, rank=0, nccl_id=None, backend=BackendKind.CudaSpectral, memory_cap_bytes=0):
        if not (kappa_u > 0.0 and kappa_v > 0.0):
            raise ConfigError("component diffusivities must be positive")
        self.kappa_u, self.kappa_v = float(kappa_u), float(kappa_v)
        super().__init__(grid, tau, family, (kappa_u, kappa_v), q, source, device, world_size, rank, nccl_id,
                         backend, memory_cap_bytes)


def make_plan(grid: Grid, tau: float, kappa: float, q: float, scheme=PadeFamily.P02,
              backend: BackendKind = BackendKind.CudaSpectral, memory_cap_bytes: int = 0,
              source: Optional[DeviceSource] = None, device: int = 0) -> StepperPlan:
    """stepper.hpp:59-61.  Spectral / CudaSpectral: eigenbasis transforms on the
    tensor cores; Thomas / CudaThomas: per-pole complex tridiagonal solves
    (thomas.cpp); ExactExpReference: the reference's exact-exponential step
    (stepper.cpp:259-295) on the spectral transforms."""
    if backend == BackendKind.ExactExpReference:
        return StepperPlan(grid, tau, kappa, q, EXACT_FAMILY, source, device, memory_cap_bytes=memory_cap_bytes)
    if backend not in _DEVICE_BACKEND:
        raise ConfigError("this package implements the Spectral, Thomas and ExactExpReference backends")
    return StepperPlan(grid, tau, kappa, q, scheme, source, device, backend=backend,
                       memory_cap_bytes=memory_cap_bytes)


def make_system_plan(grid: Grid, tau: float, kappa_u: float, kappa_v: float, q: float, scheme=PadeFamily.P02,
                     backend: BackendKind = BackendKind.CudaSpectral, source: Optional[DeviceSource] = None,
                     device: int = 0) -> SystemPlan:
    """stepper.hpp:107-108, extended to 3D (the reference throws for dim != 2).
    Spectral and Thomas backends (system_stepper.cpp:47-68)."""
    if backend not in _DEVICE_BACKEND:
        raise ConfigError("system plans support the spectral and thomas backends only")
    return SystemPlan(grid, tau, kappa_u, kappa_v, q, scheme, source, device, backend=backend)


@dataclass
class StepperState:
    """stepper.hpp:63-67 (U is x-fastest, any shape with n^dim entries)."""
    n: int = 0
    t: float = 0.0
    U: np.ndarray = field(default_factory=lambda: np.zeros(0))


@dataclass
class SystemState:
    """stepper.hpp:110-114"""
    n: int = 0
    t: float = 0.0
    U: np.ndarray = field(default_factory=lambda: np.zeros(0))
    V: np.ndarray = field(default_factory=lambda: np.zeros(0))


def advance(plan: StepperPlan, state: StepperState, f: DeviceSource, nsteps: int = 1) -> StepperState:
    """stepper.cpp:318-331 value semantics: returns a NEW state; `state` is untouched.
    nsteps > 1 is the batched extension (device-resident between steps)."""
    if not isinstance(plan, StepperPlan):
        raise ConfigError("advance needs a scalar plan")
    plan.set_source(f)
    shape = np.shape(state.U)
    u_in = np.ascontiguousarray(state.U, dtype=np.float64).reshape(-1)
    if u_in.size != plan.local_count:
        raise ConfigError("state shape does not match plan grid")
    u_out = np.empty_like(u_in)
    n, t = plan.advance_ptr(u_in.ctypes.data, 0, u_out.ctypes.data, 0, state.n, state.t, nsteps)
    return StepperState(n, t, u_out.reshape(shape))


def etd2rkds_step_2d(plan: StepperPlan, state: StepperState, f: DeviceSource) -> StepperState:
    """stepper.cpp:182-229 (one step; `advance` dispatches here for 2D plans)."""
    if not isinstance(plan, StepperPlan) or plan.grid.dim != 2:
        raise ConfigError("2D step on non-2D plan")
    if plan.family == EXACT_FAMILY:
        raise ConfigError("2D split step requires the spectral or thomas backend")
    return advance(plan, state, f)


def etd2rkds_step_3d(plan: StepperPlan, state: StepperState, f: DeviceSource) -> StepperState:
    """stepper.cpp:233-257"""
    if not isinstance(plan, StepperPlan) or plan.grid.dim != 3:
        raise ConfigError("3D step on non-3D plan")
    if plan.family == EXACT_FAMILY:
        raise ConfigError("3D split step requires the spectral or thomas backend")
    return advance(plan, state, f)


def etd2rkds_reference_step(plan: StepperPlan, state: StepperState, f: DeviceSource) -> StepperState:
    """stepper.cpp:259-295: the exact-exponential step (plans made with
    BackendKind.ExactExpReference)."""
    if not isinstance(plan, StepperPlan) or plan.family != EXACT_FAMILY:
        raise ConfigError("reference step requires the exact backend")
    return advance(plan, state, f)


def etd2rk_nonsplit_step(plan, state, f):
    """stepper.cpp:297-316: BackendKind.NonSplitBanded is not implemented on the
    device (make_plan refuses it), so no plan can take this step."""
    raise ConfigError("non-split step requires the nonsplit backend")


def phi1(x: float) -> float:
    """stepper.cpp:38-41: (1 - e^{-x})/x, series below x = 1e-4."""
    return float(lib().etd_setup_phi(1, float(x)))


def phi2(x: float) -> float:
    """stepper.cpp:43-46: (x - 1 + e^{-x})/x^2, series below x = 1e-4."""
    return float(lib().etd_setup_phi(2, float(x)))


def etd2rkds_step_system(plan: SystemPlan, state: SystemState, f: DeviceSource, nsteps: int = 1) -> SystemState:
    """system_stepper.cpp:74-114 (2D and 3D)."""
    if not isinstance(plan, SystemPlan):
        raise ConfigError("etd2rkds_step_system needs a system plan")
    if np.size(state.U) != np.size(state.V):
        raise ConfigError("system state shape does not match plan grid")
    plan.set_source(f)
    shape = np.shape(state.U)
    u_in = np.ascontiguousarray(state.U, dtype=np.float64).reshape(-1)
    v_in = np.ascontiguousarray(state.V, dtype=np.float64).reshape(-1)
    if u_in.size != plan.local_count:
        raise ConfigError("system state shape does not match plan grid")
    u_out, v_out = np.empty_like(u_in), np.empty_like(v_in)
    n, t = plan.advance_ptr(u_in.ctypes.data, v_in.ctypes.data, u_out.ctypes.data, v_out.ctypes.data, state.n,
                            state.t, nsteps)
    return SystemState(n, t, u_out.reshape(shape), v_out.reshape(shape))


# ----------------------------------------------------------------- host setup exports
def setup_axis(n: int, kappa: float, q: float, dim: int, low: float = 0.0, high: float = 1.0):
    """operators.cpp:11-56 on the host: (P column-major, lambda)."""
    P = np.empty(n * n)
    lam = np.empty(n)
    _raise(lib().etd_setup_axis(n, low, high, dim, kappa, q, _ptr(P), _ptr(lam)), None)
    return P, lam


def setup_dvector(lam: np.ndarray, tau: float, family: int, ell: int) -> np.ndarray:
    lam = np.ascontiguousarray(lam, dtype=np.float64)
    d = np.empty_like(lam)
    _raise(lib().etd_setup_dvector(lam.size, _ptr(lam), tau, int(family), ell, _ptr(d)), None)
    return d


def setup_scheme(family: int) -> np.ndarray:
    out = np.zeros(24)
    nt = C.c_int()
    _raise(lib().etd_setup_scheme(int(family), _ptr(out), C.byref(nt)), None)
    return out[: 12 * nt.value].reshape(3, nt.value, 4)


def plan_device_bytes(grid: Grid, nspecies: int = 1, world_size: int = 1, rank: int = 0,
                      backend: BackendKind = BackendKind.CudaSpectral) -> int:
    """Device bytes a plan allocates on `rank` (etd_plan_device_bytes; host only):
    the per-rank budget etd_create checks before allocating (MemoryGuardError)."""
    src = allen_cahn_cubic() if nspecies == 1 else fhn_cubic()
    kap = (1.0,) if nspecies == 1 else (1.0, 1.0)
    d = _make_desc(grid, 1.0, 0, nspecies, kap, 0.0, src, 0, world_size, rank, None, _DEVICE_BACKEND[backend])
    out = C.c_ulonglong()
    _raise(lib().etd_plan_device_bytes(C.byref(d), C.byref(out)), None)
    return out.value


def zslab_partition(n: int, world_size: int, rank: int):
    """Balanced [lo, hi) split used for z planes (x/y stages) and y rows (z stage)."""
    lo, hi = C.c_int(), C.c_int()
    _raise(lib().etd_zslab_partition(n, world_size, rank, C.byref(lo), C.byref(hi)), None)
    return lo.value, hi.value


def nccl_unique_id() -> bytes:
    """128-byte ncclUniqueId (rank 0 creates it, the others receive it out of band)."""
    buf = C.create_string_buffer(128)
    _raise(lib().etd_nccl_unique_id(C.cast(buf, C.c_void_p)), None)
    return buf.raw


def group_step(plans, nsteps: int = 1) -> None:
    """Step virtual ranks (plans created with world_size=G, rank=r, no NCCL id, one
    device) in lock-step: the sharded schedule with exchanges as device copies."""
    arr = (C.c_void_p * len(plans))(*[p.handle for p in plans])
    _raise(lib().etd_group_step(arr, len(plans), int(nsteps)), plans[0].handle)


def fill_config_ic(config: int, seed: int, species: int, n: int, z0: int = 0, z1: Optional[int] = None,
                   out: Optional[np.ndarray] = None) -> np.ndarray:
    """Seeded BASELINE initial condition, x-fastest slab [z0,z1)."""
    dim = 2 if config <= 1 else 3
    if z1 is None:
        z1 = n if dim == 3 else 1
    cnt = n * n * (z1 - z0 if dim == 3 else 1)
    a = np.empty(cnt) if out is None else out
    _raise(lib().etd_fill_config_ic(config, seed, species, n, z0, z1, _ptr(a)), None)
    return a
