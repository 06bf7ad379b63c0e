#!/bin/bash
# Build experiment variants of libparsa_b200.so (benchmark kernel only) into
# build/variants/<name>/libparsa_b200.so.  Usage: build_variants.sh name "FLAGS" ...
set -e
# needs build/obj/nelder_mead.o from the regular build (make -C paper_2408_00018_b200/csrc)
ROOT=$(cd "$(dirname "$0")/.." && pwd)
CS=$ROOT/paper_2408_00018_b200/csrc
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -prec-div=true -prec-sqrt=true -Xcompiler -fPIC -I$ROOT/include -I$CS -DPSA_EXPERIMENT_ONLY"
while [ $# -gt 1 ]; do
  name=$1; flags=$2; shift 2
  out=$ROOT/gpu_variants/$name; mkdir -p $out
  ( $NV $flags -c $CS/engine.cu -o $out/engine.o && $NV $flags -c $CS/engine_fam_schwefel_f32.cu -o $out/f32.o && \
    $NV $flags -c $CS/engine_fam_schwefel_f64.cu -o $out/f64.o && $NV $flags -c $CS/capi.cu -o $out/capi.o && \
    $NV -gencode arch=compute_100a,code=sm_100a -shared -o $out/libparsa_b200.so $out/engine.o $out/f32.o $out/f64.o $out/capi.o $ROOT/build/obj/nelder_mead.o && echo "built $name" ) &
done
wait
