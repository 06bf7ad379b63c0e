cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:v0_kernel -c 1 -o gpurun_out/s33_v0 -f python scripts/v0_run.py > gpurun_out/s29_ncu.log 2>&1; echo ncu=$?
tail -2 gpurun_out/s29_ncu.log
