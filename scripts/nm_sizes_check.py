import ctypes as C, sys, numpy as np
sys.path.insert(0,'tests'); sys.path.insert(0,'.')
from oracle_lib import Problem, oracle
from paper_2408_00018_b200 import _abi
lib=_abi.load_library()
for n in [int(a) for a in sys.argv[1:]]:
    prob=Problem("SCHWEFEL", n, -512., 512.)
    x0=np.array([400.0+ (k%13) for k in range(n)])
    cfg=_abi.psa_nm_config(1.0,2.0,0.5,0.5,1e-12,1e-10,300,0)
    xb=np.zeros(n); r=_abi.psa_nm_result(xb.ctypes.data_as(C.POINTER(C.c_double)),0,0,0,0)
    rc=lib.psa_nelder_mead_minimize(C.byref(prob.c), x0.ctypes.data_as(C.POINTER(C.c_double)), C.byref(cfg), C.byref(r))
    xo=np.zeros(n); ro=_abi.psa_nm_result(xo.ctypes.data_as(C.POINTER(C.c_double)),0,0,0,0)
    oracle().orc_nelder_mead_minimize(C.byref(prob.c), x0.ctypes.data_as(C.POINTER(C.c_double)), C.byref(cfg), C.byref(ro))
    print(n, rc, lib.psa_last_error() if rc else b'', r.f_best==ro.f_best, np.array_equal(xb.view(np.uint64), xo.view(np.uint64)), r.iterations, ro.iterations, flush=True)
    if rc: break
