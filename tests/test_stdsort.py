"""The pair form of the libstdc++ introsort restatement (used by the device
Nelder-Mead's exact sort) orders tie-heavy inputs exactly like the id form
(parsa_stdsort.h, shared with the oracle) and like std::sort itself."""
import os
import subprocess
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_pair_introsort_matches_std_sort():
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "sp")
        subprocess.run(["g++", "-std=c++17", "-O2", "-I" + os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "tests", "cxx", "stdsort_pairs_check.cpp"), "-o", exe], check=True)
        p = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "0 mismatches" in p.stdout
