"""The C++ host API (include/etdrd_b200/stepper.hpp, reference-shaped) compiles
on CPU and, on a B200, reproduces the reference golden fixtures and the
reference error semantics."""
import os
import shutil
import subprocess

import numpy as np
import pytest

from oracle import rel_gap

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "cpp_api_demo.cpp")
LIBDIR = os.path.join(ROOT, "paper_2601_06849_b200")
GOLD = os.path.join(ROOT, "tests", "golden")


def build(tmp_path):
    gxx = shutil.which("g++")
    if not gxx:
        pytest.skip("g++ unavailable")
    exe = str(tmp_path / "cpp_api_demo")
    r = subprocess.run([gxx, "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), SRC, "-o", exe,
                        os.path.join(LIBDIR, "libetd_b200.so"), f"-Wl,-rpath,{LIBDIR}"], capture_output=True,
                       text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_cpp_api_compiles(tmp_path):
    assert os.path.exists(build(tmp_path))


@pytest.mark.gpu
def test_cpp_api_errors(tmp_path):
    exe = build(tmp_path)
    r = subprocess.run([exe, "errors"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["scalar2d_p02", "scalar3d_p04", "system2d_fhn", "system3d_fhn"])
def test_cpp_api_matches_golden(tmp_path, name):
    exe = build(tmp_path)
    c = np.load(os.path.join(GOLD, name + ".npz"))
    kind = str(c["kind"])
    inp, out = str(tmp_path / "in.bin"), str(tmp_path / "out.bin")
    if kind == "scalar":
        c["u0"].astype(np.float64).tofile(inp)
        args = [kind, c["dim"], c["n"], c["tau"], c["kappa"], 0.0, c["q"], c["family"], c["steps"]]
    else:
        np.concatenate([c["u0"], c["v0"]]).tofile(inp)
        args = [kind, c["dim"], c["n"], c["tau"], c["ku"], c["kv"], c["q"], c["family"], c["steps"]]
    r = subprocess.run([exe, *[repr(float(a)) if isinstance(a, (float, np.floating)) else str(a) for a in args],
                        inp, out], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    got = np.fromfile(out)
    N = c["u0"].size
    assert rel_gap(c["u"], got[:N]) <= 1e-11
    if kind == "system":
        assert rel_gap(c["v"], got[N:]) <= 1e-11
