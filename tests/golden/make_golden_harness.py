"""Generate tests/golden/harness/* with the REFERENCE study harness itself
(oracle/_ref/libetdrd_ref.so built with harness.cpp; run_convergence,
harness.cpp:305-362): the ETRJ reference-trajectory cache files and the
convergence CSVs for two small problems without a closed-form solution.

Run in the build container (needs oracle/_ref):  python tests/golden/make_golden_harness.py
"""
import ctypes as C
import os
import shutil
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import REF_SO, Ref  # noqa: E402

# (problem, m subintervals, Ns, family, coarse)
CASES = [("singular-source-2d", 16, (16, 32), 0, 16), ("fhn-2d", 16, (16, 32), 0, 16),
         ("singular-source-3d", 8, (10, 20), 1, 10)]


def main():
    Ref.set_threads(1)
    L = C.CDLL(REF_SO)
    dst = os.path.join(HERE, "harness")
    os.makedirs(dst, exist_ok=True)
    for problem, m, Ns, fam, coarse in CASES:
        with tempfile.TemporaryDirectory() as out:
            arr = (C.c_int * len(Ns))(*Ns)
            E = (C.c_double * len(Ns))()
            err = C.create_string_buffer(256)
            rc = L.ref_run_convergence(problem.encode(), m, arr, len(Ns), fam, 0, coarse, C.c_double(0.0),
                                       out.encode(), E, err, 256)
            assert rc == 0, err.value
            for root, _, files in os.walk(out):
                for f in files:
                    if f.endswith((".traj", ".csv")):
                        shutil.copy(os.path.join(root, f), os.path.join(dst, f))
                        print(f, list(E))


if __name__ == "__main__":
    main()
