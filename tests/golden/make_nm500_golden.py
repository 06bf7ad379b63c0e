"""Large-n Nelder-Mead fixture from the UNMODIFIED reference (oracle/_ref).

Schwefel n=500 (configs[3] of BASELINE.json is the n=500 hybrid), started
from a deterministic near-optimal point and capped at 5000 iterations (the
reference needs ~0.65 ms per iteration at this n).  Exercises the device
NM's incremental centroid / diameter bookkeeping over many replacements,
expansions, contractions and new-best insertions.

    make -C oracle && python tests/golden/make_nm500_golden.py
"""
import ctypes as C
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_lib import Problem, ref  # noqa: E402

from paper_2408_00018_b200 import _abi  # noqa: E402


def main():
    n, iters = 500, 5000
    x0 = np.array([420.968746 - 60.0 + 120.0 * ((k * 37) % 101) / 100.0 for k in range(n)])
    prob = Problem("SCHWEFEL", n, -512.0, 512.0)
    nmc = _abi.psa_nm_config(1.0, 2.0, 0.5, 0.5, 1e-12, 1e-10, iters, 0)
    xb = np.zeros(n)
    r = _abi.psa_nm_result(xb.ctypes.data_as(C.POINTER(C.c_double)), 0, 0, 0, 0)
    assert ref().ref_nelder_mead(C.byref(prob.c), x0.ctypes.data_as(C.POINTER(C.c_double)), C.byref(nmc),
                                 C.byref(r)) == 0
    out = {"generator": "tests/golden/make_nm500_golden.py", "family": "SCHWEFEL", "dim": n, "lo": -512.0,
           "hi": 512.0, "max_iters": iters, "x0": [float(v).hex() for v in x0],
           "x_best": [float(v).hex() for v in xb], "f_best": float(r.f_best).hex(), "iterations": r.iterations,
           "evaluations": r.evaluations}
    with open(os.path.join(HERE, "nm500_golden.json"), "w") as fh:
        json.dump(out, fh)
    print("f_best", r.f_best, "iterations", r.iterations, "evaluations", r.evaluations)


if __name__ == "__main__":
    main()
