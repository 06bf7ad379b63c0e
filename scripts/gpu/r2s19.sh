# configs[3] end to end at the reference's default NM cap (25M iterations)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,clocks_throttle_reasons.active --format=csv > gpurun_out/s19_clocks_before.csv
timeout 3500 python scripts/c4_full.py > gpurun_out/s19_c4_full.json 2> gpurun_out/s19_c4_full.err; echo rc=$?
cat gpurun_out/s19_c4_full.json; tail -3 gpurun_out/s19_c4_full.err
