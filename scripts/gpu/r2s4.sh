# deferred-fold kernel: full GPU suite (incl. C3/C4 full-size goldens) + bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_lazy.py -q > gpurun_out/s4_lazy.log 2>&1; echo lazy_rc=$?
tail -30 gpurun_out/s4_lazy.log
timeout 900 python bench.py --no-configs --no-companion > gpurun_out/s4_bench.json 2> gpurun_out/s4_bench.err; echo bench_rc=$?
python -c "
import json;d=json.loads(open('gpurun_out/s4_bench.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['roofline']['kernel'], d.get('parity'))"
tail -5 gpurun_out/s4_bench.err
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/s4_pytest.log 2>&1; echo pytest_rc=$?
tail -30 gpurun_out/s4_pytest.log
