"""CPU: the C-ABI library loads, exports every symbol include/etd_b200.h declares,
validates configurations, refuses to run without a GPU (no CPU fallback), and
the host-side setup math matches the reference (golden)."""
import os
import re

import numpy as np
import pytest

import paper_2601_06849_b200 as etd
from oracle import rel_gap

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "etd_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(etd_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = etd.lib()
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(L, s), s
    assert L.etd_abi_version() == 4


def test_header_is_plain_c_and_matches_ctypes_layout():
    """include/etd_b200.h compiles as C99 (a C/cgo/FFI client can include it) and
    sizeof/offsetof(etd_desc) agree with the ctypes mirror in etd.py."""
    import shutil
    import subprocess
    import tempfile
    import ctypes
    cc = shutil.which("gcc")
    if not cc:
        pytest.skip("gcc unavailable")
    d = etd.etd._Desc
    fields = [f[0] for f in d._fields_]
    prog = '#include <stdio.h>\n#include <stddef.h>\n#include "etd_b200.h"\nint main(void){printf("%zu", sizeof(etd_desc));'
    for f in fields:
        prog += 'printf(" %zu", offsetof(etd_desc, ' + f + '));'
    prog += 'return 0;}\n'
    with tempfile.TemporaryDirectory() as td:
        src, exe = os.path.join(td, "h.c"), os.path.join(td, "h")
        open(src, "w").write(prog)
        subprocess.run([cc, "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), src, "-o", exe],
                       check=True)
        got = [int(x) for x in subprocess.run([exe], capture_output=True, text=True, check=True).stdout.split()]
    assert got[0] == ctypes.sizeof(d)
    assert got[1:] == [getattr(d, f).offset for f in fields]


def test_sass_targets_sm100a():
    """The extension is built for sm_100a only and uses DMMA + TMA."""
    import shutil
    import subprocess
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump unavailable")
    out = subprocess.run([exe, "-sass", etd.etd.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "DMMA.8x8x4" in out and "UTMALDG" in out


def test_config_errors_before_device():
    g = etd.unit_box_grid(2, 8)
    with pytest.raises(etd.ConfigError):
        etd.make_plan(g, 0.0, 1.0, 1.0)
    with pytest.raises(etd.ConfigError):
        etd.make_plan(g, 0.01, -1.0, 1.0)
    with pytest.raises(etd.ConfigError):
        etd.make_system_plan(g, 0.01, 1.0, 0.0, 0.0)
    with pytest.raises(etd.ConfigError):
        etd.make_plan(g, 0.01, 1.0, 1.0, source=etd.fhn_cubic())  # pair source on a scalar plan
    with pytest.raises(etd.ConfigError):
        etd.make_plan(g, 0.01, 1.0, 1.0, backend=etd.BackendKind.NonSplitBanded)
    with pytest.raises(etd.ConfigError):
        etd.make_system_plan(g, 0.01, 1.0, 1.0, 0.0, backend=etd.BackendKind.ExactExpReference)
    with pytest.raises(etd.ConfigError):
        etd.build_grid(2, [(0, 1), (1, 1)], [4, 4])
    with pytest.raises(etd.ConfigError):
        etd.unit_box_grid(3, 1)


def test_no_cpu_fallback_without_gpu():
    import ctypes
    try:
        cu = ctypes.CDLL("libcuda.so.1")
        n = ctypes.c_int(0)
        if cu.cuInit(0) == 0 and cu.cuDeviceGetCount(ctypes.byref(n)) == 0 and n.value > 0:
            pytest.skip("GPU present")
    except OSError:
        pass
    with pytest.raises(etd.DeviceError):
        etd.make_plan(etd.unit_box_grid(2, 8), 0.01, 1.0, 1.0)


def test_host_setup_matches_reference_golden():
    s = np.load(os.path.join(GOLD, "setup.npz"))
    for key in [k for k in s.files if k.startswith("P_")]:
        _, n, dim = key.split("_")
        n, dim = int(n), int(dim)
        _, _, kappa, q = s[f"diag_off_{n}_{dim}"]
        P, lam = etd.setup_axis(n, kappa, q, dim)
        assert np.array_equal(P, s[key])                       # identical closed form
        assert np.max(np.abs(lam - s[f"lam_{n}_{dim}"])) <= 1e-15 * np.max(lam)
        for fam in (0, 1):
            for ell in (1, 2, 3):
                d = etd.setup_dvector(s[f"lam_{n}_{dim}"], 0.01, fam, ell)
                assert rel_gap(s[f"d_{n}_{dim}_{fam}_{ell}"], d) <= 1e-14
    for fam in (0, 1):
        assert np.max(np.abs(etd.setup_scheme(fam) - s[f"scheme_{fam}"])) <= 1e-15


def test_config_ic_deterministic_and_slab_consistent():
    from paper_2601_06849_b200 import configs
    a = etd.fill_config_ic(3, 5, 0, 21)
    b = etd.fill_config_ic(3, 5, 0, 21)
    assert np.array_equal(a, b)
    full = a.reshape(21, 21, 21)
    part = etd.fill_config_ic(3, 5, 0, 21, 7, 13).reshape(6, 21, 21)
    assert np.array_equal(full[7:13], part)
    c = etd.fill_config_ic(3, 6, 0, 21)
    assert not np.array_equal(a, c)
    # u0 = (0.5 + 0.1 N) * S: mean of u0/S ~ 0.5, std ~ 0.1
    x = np.sin(np.pi * np.arange(1, 22) / 22)
    S = x[:, None, None] * x[None, :, None] * x[None, None, :]
    r = full / S
    assert abs(r.mean() - 0.5) < 0.01 and abs(r.std() - 0.1) < 0.01
    v = etd.fill_config_ic(3, 5, 1, 21).reshape(21, 21, 21) / S
    assert abs(v.mean()) < 0.01 and abs(v.std() - 0.1) < 0.01
    u0 = configs.initial_state(configs.CONFIGS[0], 31)[0].reshape(31, 31)
    assert np.all(np.isfinite(u0)) and abs(u0.max()) < 3.0


def test_phi_functions_match_reference_expressions():
    """stepper.cpp:38-46 (host exports, no GPU needed)."""
    import math
    for x in (0.0, 5e-5, 1e-4, 0.37, 2.0, 30.0):
        p1 = 1.0 - x / 2.0 + x * x / 6.0 - x * x * x / 24.0 if x < 1e-4 else (1.0 - math.exp(-x)) / x
        p2 = 0.5 - x / 6.0 + x * x / 24.0 - x * x * x / 120.0 if x < 1e-4 else (x - 1.0 + math.exp(-x)) / (x * x)
        assert etd.phi1(x) == p1 and etd.phi2(x) == p2


def test_step_entry_points_reject_wrong_plans():
    with pytest.raises(etd.ConfigError):
        etd.etd2rk_nonsplit_step(None, None, None)
    with pytest.raises(etd.ConfigError):
        etd.etd2rkds_step_2d(None, None, None)
