"""Study-harness loops over the device stepper (reference harness.cpp:157-421).

The reference's convergence study drives `advance` from host loops and copies a
snapshot Field at every coarse time.  Here the state stays device-resident
between snapshots (`plan.step(stride)`), and only the coarse snapshots come
back to the host.  Kept: names, argument meaning, error behaviour
(ConfigError for non-multiple N, StepperAbort re-raised with [N=...]), the
E / EOC definitions, the "ETRJ" reference-trajectory cache with its JSON
fingerprint (harness.cpp:49-115, 135-149, 246-283) and the convergence CSV and
manifest files (harness.cpp:285-301, 364-421), byte-compatible with the
reference's.  Problems are the catalogue problems with a device source
(problems.cpp:68-198): allen-cahn-2d/3d with the manufactured forcing and exact
solution, singular-source-2d/3d, fhn-2d.
"""
from __future__ import annotations

import json
import math
import os
import struct
import time
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import etd


@dataclass
class ProblemParams:
    """problems.hpp:16-26"""
    lam: float = 1.0        # decay rate of the manufactured solution ("lambda")
    rho: float = 0.1        # singular source strength
    kappa: float = 1.0      # scalar diffusivity
    sigma: float = 0.05     # Gaussian bump width
    alpha: float = 1.0      # inhibitor relaxation
    eps: float = 1.0        # activator->inhibitor coupling
    kappa_u: float = 0.01
    kappa_v: float = 10.0
    T: Optional[float] = None


@dataclass
class ProblemSpec:
    """problems.hpp:28-52 (the subset the device backend needs)."""
    name: str
    dim: int
    kappa: float = 1.0
    kappa_u: float = 0.0
    kappa_v: float = 0.0
    q: float = 0.0
    T: float = 1.0
    default_m: int = 512
    coarse: int = 16
    system: bool = False
    source: Optional[etd.DeviceSource] = None
    lam: float = 1.0
    has_exact: bool = False
    reference_N: int = 0
    sigma: float = 0.05

    def interior(self, m: int) -> int:
        return m - 1

    def initial(self, grid: etd.Grid):
        """sine_product(g, 1.0) for Allen-Cahn (problems.cpp:17-33,84), 0.99 x for
        singular (:120), the Gaussian bump for fhn-2d (:151-160)."""
        if self.system:
            return gaussian_bump(grid, self.sigma)
        return sine_product(grid, 0.99 if self.name.startswith("singular") else 1.0)

    def initial_v(self, grid: etd.Grid):
        """problems.cpp:161: V(0) = 0."""
        return np.zeros(grid.total_interior())

    def exact_field(self, grid: etd.Grid, t: float) -> np.ndarray:
        """problems.cpp:55-65 / 85-89: e^{-lambda t} prod sin(pi x_a)."""
        if not self.has_exact:
            raise etd.ConfigError(self.name + " has no closed-form solution")
        return math.exp(-self.lam * t) * sine_product(grid)


def sine_product(grid: etd.Grid, amplitude: float = 1.0) -> np.ndarray:
    """problems.cpp:17-33, same operation order: ((amp sx) sy) sz."""
    s = [np.array([math.sin(math.pi * grid.coord(a, i)) for i in range(grid.interior_shape()[a])])
         for a in range(grid.dim)]
    f = (amplitude * s[0])[None, :] * s[1][:, None]
    if grid.dim == 3:
        f = f[None, :, :] * s[2][:, None, None]
    return f.ravel()


def gaussian_bump(grid: etd.Grid, sigma: float) -> np.ndarray:
    """problems.cpp:151-160: exp(-((x-1/2)^2 + (y-1/2)^2) / sigma^2)."""
    nx, ny, _ = grid.interior_shape()
    dx = np.array([grid.coord(0, i) - 0.5 for i in range(nx)])
    dy = np.array([grid.coord(1, j) - 0.5 for j in range(ny)])
    s2 = sigma * sigma
    return np.exp(-(dx[None, :] * dx[None, :] + dy[:, None] * dy[:, None]) / s2).ravel()


def allen_cahn(dim: int, lam: float = 1.0, kappa: float = 1.0, T: float = 1.0) -> ProblemSpec:
    """problems.cpp:68-106"""
    if dim not in (2, 3):
        raise etd.ConfigError("allen-cahn: dim must be 2 or 3")
    return ProblemSpec(f"allen-cahn-{dim}d", dim, kappa=kappa, q=0.0, T=T, default_m=512 if dim == 2 else 80,
                       coarse=16 if dim == 2 else 10, source=etd.allen_cahn_manufactured(dim, lam, kappa), lam=lam,
                       has_exact=True)


def singular_source(dim: int, rho: float = 0.1, kappa: float = 1.0, T: float = 1.0) -> ProblemSpec:
    """problems.cpp:108-136"""
    if dim not in (2, 3):
        raise etd.ConfigError("singular-source: dim must be 2 or 3")
    return ProblemSpec(f"singular-source-{dim}d", dim, kappa=kappa, q=1.0, T=T, default_m=512 if dim == 2 else 80,
                       coarse=16 if dim == 2 else 10, source=etd.singular(rho),
                       reference_N=512 if dim == 2 else 320)


def fhn(kappa_u: float = 0.01, kappa_v: float = 10.0, eps: float = 1.0, alpha: float = 1.0, sigma: float = 0.05,
        T: float = 1.0) -> ProblemSpec:
    """problems.cpp:138-175: fu = u - u^3/3 - v, fv = eps (u - alpha v)."""
    return ProblemSpec("fhn-2d", 2, kappa_u=kappa_u, kappa_v=kappa_v, q=0.0, T=T, default_m=512, coarse=16,
                       system=True, source=etd.fhn_classic(eps, alpha), reference_N=512, sigma=sigma)


def problem_by_name(name: str, p: Optional[ProblemParams] = None) -> ProblemSpec:
    """problems.cpp:177-184"""
    p = p or ProblemParams()
    T = 1.0 if p.T is None else p.T
    if name in ("allen-cahn-2d", "allen-cahn-3d"):
        return allen_cahn(int(name[-2]), p.lam, p.kappa, T)
    if name in ("singular-source-2d", "singular-source-3d"):
        return singular_source(int(name[-2]), p.rho, p.kappa, T)
    if name == "fhn-2d":
        return fhn(p.kappa_u, p.kappa_v, p.eps, p.alpha, p.sigma, T)
    raise etd.ConfigError(f"unknown problem '{name}'")


def problem_names() -> List[str]:
    return ["allen-cahn-2d", "allen-cahn-3d", "singular-source-2d", "singular-source-3d", "fhn-2d"]


@dataclass
class Trajectory:
    """harness.hpp:36-40"""
    times: List[float] = field(default_factory=list)
    fields: List[np.ndarray] = field(default_factory=list)


@dataclass
class SystemTrajectory:
    """harness.hpp:42-45"""
    times: List[float] = field(default_factory=list)
    u: List[np.ndarray] = field(default_factory=list)
    v: List[np.ndarray] = field(default_factory=list)


def _check_counts(N: int, coarse: int) -> int:
    if N <= 0 or coarse <= 0 or N % coarse != 0:
        raise etd.ConfigError(f"step count must be a positive multiple of the coarse count ({N} vs {coarse})")
    return N // coarse


def integrate_scalar(spec: ProblemSpec, plan: etd.StepperPlan, N: int, coarse: int,
                     u0: Optional[np.ndarray] = None) -> Trajectory:
    """harness.cpp:157-175: snapshots at every coarse time (t=0 included)."""
    stride = _check_counts(N, coarse)
    u = spec.initial(plan.grid) if u0 is None else np.ascontiguousarray(u0, dtype=np.float64).ravel()
    plan.set_source(spec.source)
    plan.upload(0, u, 0, 0.0)
    traj = Trajectory([0.0], [u.copy()])
    for _ in range(coarse):
        plan.step(stride)
        v, n, t = plan.download(0)
        traj.times.append(t)
        traj.fields.append(v)
    return traj


def integrate_system(spec: ProblemSpec, plan: etd.SystemPlan, N: int, coarse: int) -> SystemTrajectory:
    """harness.cpp:177-197"""
    stride = _check_counts(N, coarse)
    u, v = spec.initial(plan.grid), spec.initial_v(plan.grid)
    plan.set_source(spec.source)
    plan.upload(0, u, 0, 0.0)
    plan.upload(1, v, 0, 0.0)
    traj = SystemTrajectory([0.0], [u.copy()], [v.copy()])
    for _ in range(coarse):
        plan.step(stride)
        a, n, t = plan.download(0)
        b = plan.download(1)[0]
        traj.times.append(t)
        traj.u.append(a)
        traj.v.append(b)
    return traj


def _find_time(times, t) -> int:
    tol = 1e-9 * max(1.0, abs(t))
    return next((k for k, tt in enumerate(times) if abs(tt - t) <= tol), -1)


def compute_error_E(traj, truth) -> float:
    """harness.cpp:199-232: max over shared times of the sup-norm difference
    (both components for systems)."""
    if len(traj.times) != len(truth.times):
        raise etd.ConfigError(f"trajectory snapshot counts differ: {len(traj.times)} vs {len(truth.times)}")
    comps = ("u", "v") if isinstance(traj, SystemTrajectory) else ("fields",)
    E = 0.0
    for i, t in enumerate(traj.times):
        j = _find_time(truth.times, t)
        if j < 0:
            raise etd.ConfigError(f"no matching truth snapshot at t={t}")
        for c in comps:
            a, b = getattr(traj, c)[i], getattr(truth, c)[j]
            if a.shape != b.shape:
                raise etd.ConfigError("snapshot shape mismatch against truth")
            E = max(E, float(np.max(np.abs(a - b))))
    return E


def exact_trajectory(spec: ProblemSpec, grid: etd.Grid, coarse: int) -> Trajectory:
    """harness.cpp:234-244"""
    tr = Trajectory()
    for k in range(coarse + 1):
        tk = spec.T * k / coarse
        tr.times.append(tk)
        tr.fields.append(spec.exact_field(grid, tk))
    return tr


# ----------------------------------------------------------------- ETRJ cache
_TRAJ_MAGIC = b"ETRJ"


def fingerprint_dump(fp: dict) -> str:
    """nlohmann::json::dump() of a flat object: keys sorted, no spaces, shortest
    round-trip doubles ("1.0", "0.05")."""
    return json.dumps(fp, sort_keys=True, separators=(",", ":"))


def write_traj_file(path: str, fingerprint: dict, times: List[float], comps: List[List[np.ndarray]],
                    dim: int, shape) -> None:
    """harness.cpp:55-79: "ETRJ" u32 version 1, dim, shape[3], component count,
    snapshot count, fingerprint length + JSON, then (f64 time, fields...) records."""
    os.makedirs(os.path.dirname(path) or ".", exist_ok=True)
    fp = fingerprint_dump(fingerprint).encode()
    with open(path, "wb") as f:
        f.write(_TRAJ_MAGIC)
        f.write(struct.pack("<8I", 1, dim, *[int(s) for s in shape], len(comps), len(times), len(fp)))
        f.write(fp)
        for k, t in enumerate(times):
            f.write(struct.pack("<d", t))
            for c in comps:
                f.write(np.ascontiguousarray(c[k], dtype="<f8").tobytes())


def read_traj_file(path: str, fingerprint: dict, dim: int, shape, ncomp: int):
    """harness.cpp:81-115: (times, comps) or None on any mismatch (missing file,
    wrong fingerprint, corruption)."""
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError:
        return None
    if data[:4] != _TRAJ_MAGIC or len(data) < 36:
        return None
    ver, d, s0, s1, s2, nc, count, fplen = struct.unpack_from("<8I", data, 4)
    if ver != 1 or d != dim or [s0, s1, s2] != [int(s) for s in shape] or nc != ncomp:
        return None
    off = 36
    try:
        fp = json.loads(data[off:off + fplen].decode())
    except (UnicodeDecodeError, json.JSONDecodeError):
        return None
    if fp != fingerprint:
        return None
    off += fplen
    npts = s0 * s1 * s2
    rec = 8 + 8 * npts * ncomp
    if len(data) < off + rec * count:
        return None
    times, comps = [], [[] for _ in range(ncomp)]
    for k in range(count):
        times.append(struct.unpack_from("<d", data, off)[0])
        off += 8
        for c in range(ncomp):
            comps[c].append(np.frombuffer(data, dtype="<f8", count=npts, offset=off).copy())
            off += 8 * npts
    return times, comps


def _backend_name(backend) -> str:
    """tensor_ops.cpp:88-96 (device backends report their reference names)."""
    b = etd.BackendKind(backend)
    return {etd.BackendKind.Spectral: "spectral", etd.BackendKind.CudaSpectral: "spectral",
            etd.BackendKind.Thomas: "thomas", etd.BackendKind.CudaThomas: "thomas",
            etd.BackendKind.ExactExpReference: "exact", etd.BackendKind.NonSplitBanded: "nonsplit"}[b]


def _family_name(scheme) -> str:
    return "p04" if int(scheme) == 1 else "p02"


def param_fingerprint(spec: ProblemSpec, params: ProblemParams, coarse: int, backend) -> dict:
    """harness.cpp:135-149"""
    p = params
    return {"problem": spec.name, "T": float(spec.T), "coarse": int(coarse), "backend": _backend_name(backend),
            "lambda": float(p.lam), "rho": float(p.rho), "kappa": float(p.kappa), "sigma": float(p.sigma),
            "alpha": float(p.alpha), "eps": float(p.eps), "kappa_u": float(p.kappa_u),
            "kappa_v": float(p.kappa_v)}


def reference_path(out: str, spec: ProblemSpec, m: int, scheme) -> str:
    """harness.cpp:246-250"""
    return os.path.join(out, "references", f"{spec.name}_m{m}_N{spec.reference_N}_{_family_name(scheme)}.traj")


def _plan(spec: ProblemSpec, grid, tau, scheme, backend):
    if spec.system:
        return etd.make_system_plan(grid, tau, spec.kappa_u, spec.kappa_v, spec.q, scheme, backend=backend,
                                    source=spec.source)
    return etd.make_plan(grid, tau, spec.kappa, spec.q, scheme, backend=backend, source=spec.source)


def _integrate(spec, plan, N, coarse):
    return integrate_system(spec, plan, N, coarse) if spec.system else integrate_scalar(spec, plan, N, coarse)


def truth_trajectory(spec: ProblemSpec, m: int, coarse: int, scheme=etd.PadeFamily.P02,
                     backend=etd.BackendKind.CudaSpectral, out: Optional[str] = None,
                     params: Optional[ProblemParams] = None):
    """harness.cpp:252-283: the exact solution when the problem has one, else a
    fine-N reference run, read from / written to the ETRJ cache under `out`."""
    grid = etd.unit_box_grid(spec.dim, m)
    if spec.has_exact:
        return exact_trajectory(spec, grid, coarse)
    if spec.reference_N <= 0:
        raise etd.ConfigError(spec.name + " has neither exact solution nor reference N")
    fp = param_fingerprint(spec, params or ProblemParams(), coarse, backend)
    path = reference_path(out, spec, m, scheme) if out else None
    ncomp = 2 if spec.system else 1
    shape = grid.interior_shape()
    if path:
        got = read_traj_file(path, fp, spec.dim, shape, ncomp)
        if got is not None:
            times, comps = got
            return SystemTrajectory(times, *comps) if spec.system else Trajectory(times, comps[0])
    plan = _plan(spec, grid, spec.T / spec.reference_N, scheme, backend)
    try:
        ref = _integrate(spec, plan, spec.reference_N, coarse)
    finally:
        plan.close()
    if path:
        comps = [ref.u, ref.v] if spec.system else [ref.fields]
        write_traj_file(path, fp, ref.times, comps, spec.dim, shape)
    return ref


@dataclass
class ConvergenceRow:
    N: int
    E: float
    eoc: Optional[float]
    seconds: float


@dataclass
class ConvergenceReport:
    """harness.hpp:56-60"""
    problem: str = ""
    scheme: str = ""
    backend: str = ""
    platform: str = ""
    m: int = 0
    rows: List[ConvergenceRow] = field(default_factory=list)


def platform_string() -> str:
    """harness.cpp:31-35 (uname sysname release machine)."""
    u = os.uname()
    return f"{u.sysname} {u.release} {u.machine}"


def run_convergence(spec: ProblemSpec, m: int, Ns: List[int], scheme=etd.PadeFamily.P02,
                    coarse: Optional[int] = None, backend=etd.BackendKind.CudaSpectral,
                    out: Optional[str] = None, params: Optional[ProblemParams] = None) -> List[ConvergenceRow]:
    """harness.cpp:305-362.  E(N) against the exact solution or the (cached)
    fine-N reference; EOC row r compares rows r-1 and r under step halving.
    With `out`, writes <out>/convergence_*.csv and the manifest like the reference."""
    coarse = coarse or spec.coarse
    if not Ns:
        raise etd.ConfigError("convergence study needs a nonempty N list")
    for N in Ns:
        if N <= 0 or N % coarse != 0:
            raise etd.ConfigError(f"every N must be a positive multiple of {coarse}; got {N}")
    grid = etd.unit_box_grid(spec.dim, m)
    truth = truth_trajectory(spec, m, coarse, scheme, backend, out, params)
    rows: List[ConvergenceRow] = []
    for r, N in enumerate(Ns):
        t0 = time.time()
        plan = _plan(spec, grid, spec.T / N, scheme, backend)
        try:
            E = compute_error_E(_integrate(spec, plan, N, coarse), truth)
        except etd.StepperAbort as e:
            raise etd.StepperAbort(f"{e} [N={N}]", e.t, e.step) from None
        finally:
            plan.close()
        eoc = math.log2(rows[-1].E / E) if r > 0 and N == 2 * Ns[r - 1] and E > 0 else None
        rows.append(ConvergenceRow(N, E, eoc, time.time() - t0))
    if out:
        rep = ConvergenceReport(spec.name, _family_name(scheme), _backend_name(backend), platform_string(), m, rows)
        os.makedirs(out, exist_ok=True)
        base = f"convergence_{rep.problem}_{rep.scheme}_{rep.backend}_m{m}"
        write_convergence_csv(rep, os.path.join(out, base + ".csv"))
        write_manifest(os.path.join(out, base + ".manifest.txt"), spec, rep, coarse, params or ProblemParams())
    return rows


def _g17(x: float) -> str:
    """std::ostream << double at setprecision(17)."""
    return format(x, ".17g")


def _g6(x: float) -> str:
    """std::ostream << double at the default precision 6."""
    return format(x, "g")


def write_convergence_csv(report: ConvergenceReport, path: str) -> None:
    """harness.cpp:364-378"""
    lines = [f"# problem={report.problem} scheme={report.scheme} backend={report.backend} m={report.m} "
             f"platform={report.platform}", "N,E,EOC,cpu_seconds"]
    for r in report.rows:
        lines.append(f"{r.N},{_g17(r.E)},{'' if r.eoc is None else _g17(r.eoc)},{_g17(r.seconds)}")
    with open(path, "w") as f:
        f.write("\n".join(lines) + "\n")


def parse_convergence_csv(path: str) -> ConvergenceReport:
    """harness.cpp:380-421"""
    rep = ConvergenceReport()
    with open(path) as f:
        for line in f:
            line = line.rstrip("\n")
            if not line:
                continue
            if line.startswith("#"):
                toks = line[1:].split()
                for k, tok in enumerate(toks):
                    if "=" not in tok:
                        continue
                    key, val = tok.split("=", 1)
                    if key == "problem":
                        rep.problem = val
                    elif key == "scheme":
                        rep.scheme = val
                    elif key == "backend":
                        rep.backend = val
                    elif key == "m":
                        rep.m = int(val)
                    elif key == "platform":
                        rep.platform = " ".join([val] + toks[k + 1:])
                        break
                continue
            if line.startswith("N,"):
                continue
            N, E, eoc, sec = line.split(",")
            rep.rows.append(ConvergenceRow(int(N), float(E), float(eoc) if eoc else None, float(sec)))
    return rep


def write_manifest(path: str, spec: ProblemSpec, rep: ConvergenceReport, coarse: int, p: ProblemParams,
                   extra: str = "") -> None:
    """harness.cpp:285-301"""
    lines = [f"problem={spec.name}", f"m={rep.m}", f"scheme={rep.scheme}", f"backend={rep.backend}",
             f"T={_g6(spec.T)}", f"coarse={coarse}", f"platform={rep.platform}", f"lambda={_g6(p.lam)}",
             f"rho={_g6(p.rho)}", f"kappa={_g6(p.kappa)}", f"sigma={_g6(p.sigma)}", f"alpha={_g6(p.alpha)}",
             f"eps={_g6(p.eps)}", f"kappa_u={_g6(p.kappa_u)}", f"kappa_v={_g6(p.kappa_v)}"]
    if spec.reference_N > 0:
        lines.append(f"reference_N={spec.reference_N}")
    with open(path, "w") as f:
        f.write("\n".join(lines) + "\n" + extra)
