cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
PSA_LIB_PATH=gpu_variants/nmprof/libparsa_b200.so timeout 900 python scripts/nm_rate.py 1000000 > gpurun_out/s20_nmprof.log 2>&1; echo rc=$?
cat gpurun_out/s20_nmprof.log
timeout 900 python -m pytest tests/test_lazy.py -q -x > gpurun_out/s20_lazy.log 2>&1; echo lazy_rc=$?
tail -3 gpurun_out/s20_lazy.log
