# configs[3] end to end at the reference's default NM cap (25M iterations), round-2 final NM
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 3300 python scripts/c4_full.py > gpurun_out/s40_c4_full.json 2> gpurun_out/s40_c4_full.err; echo rc=$?
cat gpurun_out/s40_c4_full.json; tail -3 gpurun_out/s40_c4_full.err
