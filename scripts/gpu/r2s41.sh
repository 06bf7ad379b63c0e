cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_bench_parity.py -q -x -k "nelder or hybrid or nm or c4" > /tmp/t.log 2>&1; echo nmtests=$?; tail -2 /tmp/t.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
