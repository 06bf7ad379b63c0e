cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
PSA_LIB_PATH=gpu_variants/nmprof/libparsa_b200.so timeout 900 python scripts/nm_rate.py 20000 300000 3000000 > gpurun_out/s17_nmprof.log 2>&1; echo rc=$?
cat gpurun_out/s17_nmprof.log
