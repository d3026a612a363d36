"""In-tree build of the CUDA extension ``libetd_b200.so`` (sm_100a only).

``python -m paper_2601_06849_b200.build`` or ``__graft_entry__.build()``.
The shared library is written next to this file so it travels with the repo
snapshot to the GPU box (a JIT cache under ~/.cache would not).
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libetd_b200.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
SOURCES = ["etd_setup.cpp", "etd_plan.cu", "etd_specs_dense.cu", "etd_specs_fold.cu", "etd_specs_fold2.cu",
           "etd_specs_fold6.cu"]
HEADERS = ["etd_setup.hpp", "etd_kernels.cuh", "etd_thomas.cuh", "etd_registry.cuh", "etd_back6.cuh"]


def _nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False, ptxas_verbose: bool = False) -> str:
    nvcc = _nvcc()
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "etd_b200.h")]
    if not force and not _stale(LIB, deps):
        return LIB
    objdir = os.path.join(CSRC, "_obj")
    os.makedirs(objdir, exist_ok=True)
    common = ["-O3", "-std=c++20", "-Xcompiler", "-fPIC", "-I" + os.path.join(ROOT, "include")]
    common += os.environ.get("ETD_BUILD_DEFS", "").split()  # diagnostics, e.g. -DETD_CTA_TRACE_BUILD

    def compile_one(src):
        obj = os.path.join(objdir, os.path.splitext(src)[0] + ".o")
        cmd = [nvcc, *ARCH, *common, "-lineinfo", "-c", os.path.join(CSRC, src), "-o", obj]
        if src.endswith(".cu"):
            cmd += ["--expt-relaxed-constexpr"]
            if ptxas_verbose:
                cmd += ["-Xptxas", "-v"]
        if verbose:
            print(" ".join(cmd))
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{r.stdout}\n{r.stderr}")
        return obj, r.stdout + r.stderr

    # the translation units compile in parallel (the kernel variants dominate)
    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        res = list(ex.map(compile_one, SOURCES))
    objs = [o for o, _ in res]
    if verbose or ptxas_verbose:
        for _, log in res:
            sys.stdout.write(log)
    tmp = LIB + ".tmp"
    cmd = [nvcc, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv, ptxas_verbose="--ptxas" in sys.argv))
