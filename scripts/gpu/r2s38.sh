cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
./scripts/sort_probe > gpurun_out/s38_sort_probe.jsonl 2>&1; head -5 gpurun_out/s38_sort_probe.jsonl
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_bench_parity.py -q -x -k "nelder or hybrid or nm or c4" > gpurun_out/s38_nm_tests.log 2>&1; echo nmtests=$?
tail -2 gpurun_out/s38_nm_tests.log
timeout 1500 python scripts/nm_rate.py 3000000 10000000 > gpurun_out/s38_nm_rate.jsonl 2>&1; echo rc=$?
cat gpurun_out/s38_nm_rate.jsonl
