#!/bin/bash
# A/B of gpu_variants/*/libparsa_b200.so on the single-chain V2 kernel:
# C2 f32 and f64 (2^20 chains, Tmin 500) and C1/C3 per-level costs.
cd "$(dirname "$0")/.."
for d in gpu_variants/*/; do
  n=$(basename $d)
  for p in f32 f64; do
    v=$(PSA_V2_MODE=single PSA_LIB_PATH=$PWD/$d/libparsa_b200.so timeout 300 python bench.py --tmin 500 --precision $p --no-cpu-baseline --no-companion --steps 2 --warmup 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4e'%d['value'])")
    echo "$n C2-single $p $v"
  done
  PSA_LIB_PATH=$PWD/$d/libparsa_b200.so timeout 300 python scripts/level_overhead.py | sed "s/^/$n /" | cut -c1-60
done
