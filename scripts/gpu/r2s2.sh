# Round 2, session 2: full GPU suite (no -x) + default bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -k "not c3_full and not c4_hybrid_table8" -p no:randomly > gpurun_out/s2_pytest.log 2>&1; echo pytest_rc=$?
tail -40 gpurun_out/s2_pytest.log
timeout 600 python bench.py > gpurun_out/s2_bench.json 2> gpurun_out/s2_bench.err; echo bench_rc=$?
tail -c 3000 gpurun_out/s2_bench.json
