#!/bin/bash
# A/B of the device throughput: gpu_variants/<name>/libparsa_b200.so (the
# benchmark families only: C1, C2, C3 Schwefel) against the in-tree library
# (every config).  Usage: scripts/ab_configs.sh name...
cd "$(dirname "$0")/.."
for n in "$@"; do
  PSA_LIB_PATH=$PWD/gpu_variants/$n/libparsa_b200.so timeout 600 python scripts/measure_configs.py --only C1,C2 | sed "s/^/$n /"
done
timeout 900 python scripts/measure_configs.py | sed "s/^/tree /"
