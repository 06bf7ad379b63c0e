"""The device math library's glibc restatements, compiled for the host,
against this host's libm (CPU).  The exhaustive single-precision check
(every finite float; oracle/check_libm.cpp) is recorded in
profiles/libm_exhaustive_f32.txt; here a strided sample is re-checked on
every run, plus random doubles over the reference's argument ranges."""
import ctypes as C
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
libm = C.CDLL("libm.so.6")
for nm in ("sinf", "cosf", "expf"):
    getattr(libm, nm).restype = C.c_float
    getattr(libm, nm).argtypes = [C.c_float]
for nm in ("sin", "cos", "exp"):
    getattr(libm, nm).restype = C.c_double
    getattr(libm, nm).argtypes = [C.c_double]


def _f32_bits(v):
    return np.float32(v).view(np.uint32)


def test_float_restatements_strided(lib):
    rng = np.random.default_rng(0)
    bits = np.concatenate([rng.integers(0, 0x7F800000, 60000, dtype=np.uint32),
                           rng.integers(0x80000000, 0xFF800000, 60000, dtype=np.uint32)])
    xs = bits.view(np.float32)
    # targeted: the Schwefel argument range sqrt|x| in [0, 22.63] and Metropolis exponents
    xs = np.concatenate([xs, np.sqrt(rng.uniform(0, 512, 40000)).astype(np.float32),
                         -rng.exponential(5.0, 40000).astype(np.float32)])
    bad = {"sinf": 0, "cosf": 0, "expf": 0}
    for x in xs.tolist():
        for nm in bad:
            a = getattr(libm, nm)(x)
            b = getattr(lib, "psa_libm_" + nm)(x)
            if _f32_bits(a) != _f32_bits(b) and not (np.isnan(a) and np.isnan(b)):
                bad[nm] += 1
    assert bad == {"sinf": 0, "cosf": 0, "expf": 0}


def test_double_restatements_random(lib):
    rng = np.random.default_rng(1)
    ranges = [(0, 0.126), (0.126, 0.855), (0.855, 2.43), (2.43, 23.0), (23, 4000), (-30, 30)]
    bad = {"sin": 0, "cos": 0}
    for lo, hi in ranges:
        for x in rng.uniform(lo, hi, 15000).tolist():
            for nm in bad:
                if getattr(libm, nm)(x) != getattr(lib, "psa_libm_" + nm)(x):
                    bad[nm] += 1
    e = 0
    for x in np.concatenate([rng.uniform(-745, 0, 40000), rng.uniform(-1, 1, 10000), rng.uniform(0, 709, 10000)]).tolist():
        a, b = libm.exp(x), lib.psa_libm_exp(x)
        if np.float64(a).view(np.uint64) != np.float64(b).view(np.uint64):
            e += 1
    assert bad == {"sin": 0, "cos": 0} and e == 0


def test_exhaustive_record_present():
    rec = open(os.path.join(ROOT, "profiles", "libm_exhaustive_f32.txt")).read()
    assert "sinf: 0 mismatches of 4278190080" in rec
    assert "cosf: 0 mismatches of 4278190080" in rec
    assert "expf: 0 mismatches of" in rec
