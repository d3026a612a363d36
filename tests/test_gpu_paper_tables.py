"""GPU known-answer tests from the paper / reference release gates: the CUDA
path reproduces the published error tables of the manufactured Allen-Cahn
problem (reference acceptance gates 1-3, acceptance_main.cpp:526-542; PAPER.md
Tables 1-2): E(N) = max over the coarse snapshots of sup|U - u_exact| with
u_exact = e^{-t} prod sin(pi x_a), T = 1, kappa = lambda = 1, q = 0
(problems.cpp:68-106, harness.cpp:199-232).  Gate tolerance: 10% on E, 0.05
on EOC (acceptance_main.cpp:100-118)."""
import math

import numpy as np
import pytest

import paper_2601_06849_b200 as etd
from paper_2601_06849_b200 import harness

pytestmark = pytest.mark.gpu


def error_E(dim, n, N, family, coarse):
    """E(N) through the device harness (harness.cpp:305-362 semantics)."""
    spec = harness.allen_cahn(dim)
    rows = harness.run_convergence(spec, n + 1, [N], scheme=family, coarse=coarse)
    return rows[0].E


def eoc(E):
    return [math.log2(E[i - 1] / E[i]) for i in range(1, len(E))]


def test_table1_2d_p02_gate1():
    Ns = [16, 32, 64, 128, 256]
    E = [error_E(2, 511, N, 0, 16) for N in Ns]
    golden = [5.05e-2, 1.53e-2, 4.15e-3, 1.08e-3, 2.76e-4]
    for e, g in zip(E, golden):
        assert abs(e - g) / g <= 0.10, (E, golden)
    for o, g in zip(eoc(E), [1.72, 1.88, 1.94, 1.97]):
        assert abs(o - g) <= 0.05, eoc(E)


def test_table1_2d_p04_gate2():
    Ns = [16, 32, 64, 128, 256]
    E = [error_E(2, 511, N, 1, 16) for N in Ns]
    assert abs(E[-1] - 9.73e-5) / 9.73e-5 <= 0.10, E
    assert abs(eoc(E)[-1] - 2.0) <= 0.15, eoc(E)


def test_table2_3d_p02_gate3():
    Ns = [10, 20, 40, 80, 160]
    E = [error_E(3, 79, N, 0, 10) for N in Ns]
    golden = [2.96e-1, 1.04e-1, 3.01e-2, 8.05e-3, 2.14e-3]
    for e, g in zip(E, golden):
        assert abs(e - g) / g <= 0.10, (E, golden)


def test_run_convergence_eoc_and_guards():
    """run_convergence reports EOC under step halving and rejects N not a multiple
    of the coarse count (harness.cpp:307-312)."""
    spec = harness.allen_cahn(2)
    rows = harness.run_convergence(spec, 64, [32, 64, 128], coarse=16)
    assert rows[0].eoc is None and all(r.eoc is not None for r in rows[1:])
    assert all(1.5 < r.eoc < 2.5 for r in rows[1:])
    with pytest.raises(etd.ConfigError):
        harness.run_convergence(spec, 64, [24], coarse=16)
