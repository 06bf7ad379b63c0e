cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
PSA_LIB_PATH=gpu_variants/nmprof/libparsa_b200.so timeout 1800 python scripts/nm_rate.py 14000000 > gpurun_out/s37_nmprof.log 2>&1; echo rc=$?
cat gpurun_out/s37_nmprof.log
