"""Record the reference harness's report files as byte-exact fixtures.

Runs oracle/_ref/ref_harness (the UNMODIFIED reference harness.cpp +
engines, built by oracle/Makefile) on each config in HARNESS_SPECS and
stores every file it writes under tests/golden/harness/<name>/, with the
wall-time fields (the only host-dependent bytes, docs/reporting.md:5-7)
masked by mask_wall_times().  tests/test_reference_suites.py runs the B200
CLI (`parsa run --config`) on the same configs and compares byte for byte.

    make -C oracle && python tests/golden/make_harness_golden.py
"""
from __future__ import annotations

import json
import os
import re
import shutil
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
OUT = os.path.join(HERE, "harness")

# name -> JSON config (docs/reporting.md schema); output paths are relative
# to the run directory
HARNESS_SPECS = {
    "f5_v2_two_reps": {
        "function": "F5", "engine": "v2", "t0": 10, "tmin": 0.1, "rho": 0.8, "chain_length": 10,
        "chains": 32, "seed": 1, "reps": 2,
        "out": "rows.csv", "summary": "summary.json", "trace": "trace.csv",
    },
    "f0a_v1_random_single": {
        "function": "F0_a", "engine": "v1", "t0": 100, "tmin": 0.5, "rho": 0.9, "chain_length": 20,
        "chains": "16x4", "start": "random", "seed": 7, "reps": 3, "precision": "single",
        "out": "rows.csv", "summary": "summary.json", "trace": "t.csv",
    },
    "f14_hybrid": {
        "function": "F14", "engine": "hybrid", "t0": 10, "tmin": 0.1, "rho": 0.9, "chain_length": 20,
        "chains": 64, "seed": 0, "reps": 2, "nm": {"max_iters": 3000},
        "out": "rows.csv", "summary": "summary.json", "trace": "trace.csv",
    },
    "f12a_v0_unknown_location": {
        "function": "F12_a", "engine": "v0", "t0": 5, "tmin": 0.05, "rho": 0.7, "chain_length": 30,
        "chains": 1, "seed": 3, "reps": 1,
        "out": "rows.csv", "summary": "summary.json", "trace": "trace.csv",
    },
    "f9_v2_start_point": {
        "function": "F9", "engine": "v2", "t0": 50, "tmin": 0.5, "rho": 0.85, "chain_length": 15,
        "chains": 48, "start_point": [1.5, -2.25], "seed": 11, "reps": 2,
        "out": "rows.csv", "summary": "summary.json",
    },
}


def mask_wall_times(name: str, text: str) -> str:
    """Replace wall-time values (rows CSV last column, summary wall_time_s block)."""
    if name.endswith(".csv") and text.startswith("seed,best_f,value_error,location_error,evaluations,wall_time_s"):
        lines = text.split("\n")
        out = [lines[0]]
        for ln in lines[1:]:
            out.append(ln.rsplit(",", 1)[0] + ",*" if ln else ln)
        return "\n".join(out)
    if name.endswith(".json"):
        return re.sub(r'("wall_time_s": \{[^}]*\})',
                      lambda m: re.sub(r'(": )[-0-9.eE+]+', r'\1*', m.group(1)), text)
    return text


def run_reference(name: str, spec: dict) -> dict:
    exe = os.path.join(ROOT, "oracle", "_ref", "ref_harness")
    with tempfile.TemporaryDirectory() as d:
        cfg = os.path.join(d, "config.json")
        with open(cfg, "w") as fh:
            json.dump(spec, fh)
        subprocess.run([exe, "run", cfg], cwd=d, check=True, capture_output=True, text=True)
        files = {}
        for fn in sorted(os.listdir(d)):
            if fn == "config.json":
                continue
            with open(os.path.join(d, fn)) as fh:
                files[fn] = mask_wall_times(fn, fh.read())
        return files


def main() -> None:
    if os.path.isdir(OUT):
        shutil.rmtree(OUT)
    for name, spec in HARNESS_SPECS.items():
        files = run_reference(name, spec)
        dst = os.path.join(OUT, name)
        os.makedirs(dst)
        with open(os.path.join(dst, "config.json"), "w") as fh:
            json.dump(spec, fh, indent=1)
        for fn, text in files.items():
            with open(os.path.join(dst, fn), "w") as fh:
                fh.write(text)
        print(name, sorted(files))


if __name__ == "__main__":
    sys.exit(main())
