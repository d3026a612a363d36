"""Study-harness loops over the device stepper (reference harness.cpp:157-362).

The reference's convergence study drives `advance` from host loops and copies a
snapshot Field at every coarse time.  Here the state stays device-resident
between snapshots (`plan.step(stride)`), and only the coarse snapshots come
back to the host.  Kept: names, argument meaning, error behaviour
(ConfigError for non-multiple N, StepperAbort re-raised with [N=...]), and the
E / EOC definitions.  Problems are the catalogue problems with a device source
(allen-cahn-2d/3d with the manufactured forcing and exact solution,
singular-source-2d/3d, fhn-2d).
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import etd


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

    def interior(self, m: int) -> int:
        return m - 1

    def initial(self, grid: etd.Grid):
        """sine_product(g, 1.0) for Allen-Cahn (problems.cpp:17-33,84), 0.99 x for singular."""
        if self.system:
            raise etd.ConfigError("system initial data is problem specific; pass it explicitly")
        amp = 0.99 if self.name.startswith("singular") else 1.0
        return amp * sine_product(grid)

    def exact_field(self, grid: etd.Grid, t: float) -> np.ndarray:
        """problems.cpp:55-65 / 85-89: e^{-lambda t} prod sin(pi x_a)."""
        if not self.has_exact:
            raise etd.ConfigError(self.name + " has no closed-form solution")
        return math.exp(-self.lam * t) * sine_product(grid)


def sine_product(grid: etd.Grid) -> np.ndarray:
    nx, ny, nz = grid.interior_shape()
    s = [np.array([math.sin(math.pi * grid.coord(a, i)) for i in range(grid.interior_shape()[a])])
         for a in range(grid.dim)]
    f = s[0][None, :] * s[1][:, None]
    if grid.dim == 3:
        f = f[None, :, :] * s[2][:, None, None]
    return f.ravel()


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
                       coarse=16 if dim == 2 else 10, source=etd.singular(rho))


@dataclass
class Trajectory:
    """harness.hpp:36-40"""
    times: List[float] = field(default_factory=list)
    fields: List[np.ndarray] = field(default_factory=list)


def integrate_scalar(spec: ProblemSpec, plan: etd.StepperPlan, N: int, coarse: int,
                     u0: Optional[np.ndarray] = None) -> Trajectory:
    """harness.cpp:157-175: snapshots at every coarse time (t=0 included)."""
    if N <= 0 or coarse <= 0 or N % coarse != 0:
        raise etd.ConfigError(f"step count must be a positive multiple of the coarse count ({N} vs {coarse})")
    stride = N // coarse
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


def compute_error_E(traj: Trajectory, truth: Trajectory) -> float:
    """harness.cpp:199-215: max over shared times of the sup-norm difference."""
    if len(traj.times) != len(truth.times):
        raise etd.ConfigError(f"trajectory snapshot counts differ: {len(traj.times)} vs {len(truth.times)}")
    E = 0.0
    for t, f in zip(traj.times, traj.fields):
        j = next((k for k, tt in enumerate(truth.times) if abs(tt - t) <= 1e-9 * max(1.0, abs(t))), -1)
        if j < 0:
            raise etd.ConfigError(f"no matching truth snapshot at t={t}")
        if truth.fields[j].shape != f.shape:
            raise etd.ConfigError("snapshot shape mismatch against truth")
        E = max(E, float(np.max(np.abs(f - truth.fields[j]))))
    return E


def exact_trajectory(spec: ProblemSpec, grid: etd.Grid, coarse: int) -> Trajectory:
    """harness.cpp:234-244"""
    tr = Trajectory()
    for k in range(coarse + 1):
        tk = spec.T * k / coarse
        tr.times.append(tk)
        tr.fields.append(spec.exact_field(grid, tk))
    return tr


@dataclass
class ConvergenceRow:
    N: int
    E: float
    eoc: Optional[float]
    seconds: float


def run_convergence(spec: ProblemSpec, m: int, Ns: List[int], scheme=etd.PadeFamily.P02,
                    coarse: Optional[int] = None) -> List[ConvergenceRow]:
    """harness.cpp:305-362 against the exact solution (problems with has_exact).
    EOC row r compares rows r-1 and r under step halving."""
    coarse = coarse or spec.coarse
    if not Ns:
        raise etd.ConfigError("convergence study needs a nonempty N list")
    for N in Ns:
        if N <= 0 or N % coarse != 0:
            raise etd.ConfigError(f"every N must be a positive multiple of {coarse}; got {N}")
    grid = etd.unit_box_grid(spec.dim, m)
    truth = exact_trajectory(spec, grid, coarse)
    rows: List[ConvergenceRow] = []
    for r, N in enumerate(Ns):
        t0 = time.time()
        plan = etd.make_plan(grid, spec.T / N, spec.kappa, spec.q, scheme, source=spec.source)
        try:
            E = compute_error_E(integrate_scalar(spec, plan, N, coarse), truth)
        except etd.StepperAbort as e:
            raise etd.StepperAbort(f"{e} [N={N}]", e.t, e.step) from None
        finally:
            plan.close()
        eoc = math.log2(rows[-1].E / E) if r > 0 and N == 2 * Ns[r - 1] and E > 0 else None
        rows.append(ConvergenceRow(N, E, eoc, time.time() - t0))
    return rows
