"""The five BASELINE.json configurations.

BASELINE "m" counts interior points; the reference Grid::m counts subintervals
(grid.hpp:14-16), so config m=127 is unit_box_grid(dim, 128).  Pade family is
the reference default P02 (harness.hpp:23).  Initial conditions come from the
seeded counter-based generator in the extension (etd_fill_config_ic) so that
the oracle and the GPU receive identical host arrays.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import etd

SEED = 2601_06849


@dataclass(frozen=True)
class Config:
    id: int
    dim: int
    n: int
    tau: float
    steps: int
    q: float
    kappa: tuple  # (kappa,) or (kappa_u, kappa_v)
    family: int = 0

    @property
    def nspecies(self) -> int:
        return len(self.kappa)

    @property
    def source(self) -> etd.DeviceSource:
        return etd.allen_cahn_cubic() if self.nspecies == 1 else etd.fhn_cubic(0.1, 0.01, 0.5)

    def points(self, n: Optional[int] = None) -> int:
        n = self.n if n is None else n
        return n ** self.dim

    def transforms_per_step(self) -> int:
        """Algorithm 1 (2D): 9, Algorithm 2 (3D): 13 transforms per species."""
        return 9 if self.dim == 2 else 13

    def flops_per_step(self, n: Optional[int] = None) -> float:
        n = self.n if n is None else n
        return self.transforms_per_step() * 2.0 * n * self.points(n) * self.nspecies

    def describe(self) -> str:
        src = "u-u^3" if self.nspecies == 1 else "FHN u(1-u)(u-0.1)-v, 0.01(0.5u-v)"
        k = ",".join(f"{x:g}" for x in self.kappa)
        return f"cfg{self.id}: {self.dim}D n={self.n} kappa={k} q={self.q:g} tau={self.tau:g} steps={self.steps} f={src}"


CONFIGS = [
    Config(0, 2, 127, 1e-3, 100, 1.0, (1.0,)),
    Config(1, 2, 1023, 5e-4, 200, 0.0, (0.5,)),
    Config(2, 3, 255, 1e-3, 50, 1.0, (0.1,)),
    Config(3, 3, 511, 0.05, 50, 0.0, (1e-3, 5e-4)),
    Config(4, 3, 1023, 0.05, 20, 0.0, (1e-3, 5e-4)),
]


def initial_state(cfg: Config, n: Optional[int] = None, seed: int = SEED, z0: int = 0, z1: Optional[int] = None):
    """[u0] or [u0, v0] as flat x-fastest float64 arrays (slab [z0,z1) in 3D)."""
    n = cfg.n if n is None else n
    return [etd.fill_config_ic(cfg.id, seed, s, n, z0, z1) for s in range(cfg.nspecies)]


def make_plan(cfg: Config, n: Optional[int] = None, device: int = 0, **kw):
    n = cfg.n if n is None else n
    g = etd.unit_box_grid(cfg.dim, n + 1)
    if cfg.nspecies == 1:
        return etd.StepperPlan(g, cfg.tau, cfg.kappa[0], cfg.q, cfg.family, cfg.source, device, **kw)
    return etd.SystemPlan(g, cfg.tau, cfg.kappa[0], cfg.kappa[1], cfg.q, cfg.family, cfg.source, device, **kw)
