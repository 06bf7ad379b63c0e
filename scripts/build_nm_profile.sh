#!/bin/bash
# Measurement build: the library with a phase-timed Nelder-Mead kernel
# (-DPSA_NM_PROFILE: cycles per phase and path counters, printed by the
# kernel) into gpu_variants/nmprof/libparsa_b200.so; use with PSA_LIB_PATH.
# Needs the regular objects (make -C paper_2408_00018_b200/csrc).
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
CS=$ROOT/paper_2408_00018_b200/csrc
OUT=$ROOT/gpu_variants/nmprof
mkdir -p $OUT
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -prec-div=true -prec-sqrt=true -Xcompiler -fPIC -I$ROOT/include -I$CS"
$NV -DPSA_NM_PROFILE $* -c $CS/nelder_mead.cu -o $OUT/nelder_mead.o
O=$ROOT/build/obj
$NV -shared -o $OUT/libparsa_b200.so $O/engine.o $O/engine_fam_*.o $O/capi.o $OUT/nelder_mead.o
echo built $OUT/libparsa_b200.so
