cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "nelder or hybrid or nm" > gpurun_out/s22_nm_tests.log 2>&1; echo nmtests=$?
tail -3 gpurun_out/s22_nm_tests.log
timeout 900 python -m pytest tests/test_bench_parity.py -q -x -k "c4" > gpurun_out/s22_c4.log 2>&1; echo c4=$?
tail -2 gpurun_out/s22_c4.log
PSA_LIB_PATH=gpu_variants/nmprof/libparsa_b200.so timeout 900 python scripts/nm_rate.py 20000 1000000 > gpurun_out/s22_nmprof.log 2>&1; echo rc=$?
cat gpurun_out/s22_nmprof.log
