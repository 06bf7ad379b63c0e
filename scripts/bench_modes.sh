#!/bin/bash
# A/B the V2 kernel modes of every gpu_variants/<name>/libparsa_b200.so on the
# full C2 ladder (1146 levels) and on its high-temperature head (--tmin 500).
cd "$(dirname "$0")/.."
for d in gpu_variants/*/; do
  n=$(basename $d)
  for mode in ${MODES:-pair lazy}; do
    for tmin in 0.01 500; do
      v=$(PSA_V2_MODE=$mode PSA_LIB_PATH=$PWD/$d/libparsa_b200.so timeout 300 python bench.py --tmin $tmin --no-cpu-baseline --no-companion --steps 2 --warmup 3 "$@" 2>gpurun_out/variant_${n}_$mode.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4e'%d['value'])")
      echo "$n $mode tmin=$tmin $v"
    done
  done
done
