#!/bin/bash
# Bench every gpu_variants/<name>/libparsa_b200.so on the short C2 ladder.
cd "$(dirname "$0")/.."
for d in gpu_variants/*/; do
  n=$(basename $d)
  v=$(PSA_LIB_PATH=$PWD/$d/libparsa_b200.so timeout 300 python bench.py --tmin 500 --no-cpu-baseline --no-companion --steps 3 --warmup 3 "$@" 2>gpurun_out/variant_$n.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4e'%d['value'])")
  echo "$n $v"
done
