"""The C-ABI boundary: the library loads, exports every symbol the header
declares, and its struct layouts match the ctypes mirror (CPU only; no
compute calls)."""
import os
import re
import subprocess
import tempfile

import ctypes as C

import pytest

from paper_2408_00018_b200 import _abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "parsa_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(psa_[a-z0-9_]+)\s*\(", src)))


def test_library_loads_and_exports_every_declared_symbol(lib):
    decl = declared_functions()
    assert len(decl) >= 25
    assert sorted(_abi.EXPORTED_SYMBOLS) == decl
    for name in decl:
        assert hasattr(lib, name), name
    assert lib.psa_abi_version() == _abi.ABI_VERSION == 2
    out = subprocess.run(["nm", "-D", "--defined-only", _abi.LIB_PATH], capture_output=True, text=True).stdout
    for name in decl:
        assert re.search(rf"\bT {name}\b", out), name


def test_no_oracle_linkage():
    """The product library must not link or reference the CPU oracle."""
    out = subprocess.run(["ldd", _abi.LIB_PATH], capture_output=True, text=True).stdout
    assert "oracle" not in out and "parsa_ref" not in out
    syms = subprocess.run(["nm", "-D", _abi.LIB_PATH], capture_output=True, text=True).stdout
    assert "orc_" not in syms and "ref_run" not in syms


STRUCTS = {
    "psa_objective": _abi.psa_objective,
    "psa_schedule": _abi.psa_schedule,
    "psa_engine_config": _abi.psa_engine_config,
    "psa_trace_point": _abi.psa_trace_point,
    "psa_run_result": _abi.psa_run_result,
    "psa_nm_config": _abi.psa_nm_config,
    "psa_nm_result": _abi.psa_nm_result,
}


def test_struct_layouts_match_header():
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "parsa_b200.h"', "int main(void){"]
    for name, cls in STRUCTS.items():
        lines.append(f'printf("{name} %zu\\n", sizeof({name}));')
        for fname, _ in cls._fields_:
            lines.append(f'printf("{name}.{fname} %zu\\n", offsetof({name}, {fname}));')
    lines.append("return 0;}")
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "layout.c")
        exe = os.path.join(d, "layout")
        open(src, "w").write("\n".join(lines))
        subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), src, "-o", exe])
        out = subprocess.check_output([exe], text=True)
    got = dict(line.rsplit(" ", 1) for line in out.strip().splitlines())
    for name, cls in STRUCTS.items():
        assert int(got[name]) == C.sizeof(cls), name
        for fname, _ in cls._fields_:
            assert int(got[f"{name}.{fname}"]) == getattr(cls, fname).offset, (name, fname)


def test_oracle_library_exports():
    from oracle_lib import oracle
    o = oracle()
    hdr = open(os.path.join(ROOT, "oracle", "sa_oracle.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    for name in set(re.findall(r"\b(orc_[a-z0-9_]+)\s*\(", hdr)):
        assert hasattr(o, name), name


def test_engine_without_device_fails_loudly(lib):
    """No CPU fallback: with no sm_100 device the engines refuse to run."""
    if lib.psa_device_count() > 0:
        pytest.skip("a device is present")
    import paper_2408_00018_b200 as psa
    with pytest.raises(psa.DeviceError, match="no CPU fallback"):
        psa.run_synchronous(psa.registry_get("F0_a"), psa.EngineConfig(n_chains=4))
