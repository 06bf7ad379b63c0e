cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s34_smoke.log 2>&1; echo smoke=$?
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/s34_pytest.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/s34_pytest.log
timeout 900 python bench.py > gpurun_out/s34_bench.json 2> gpurun_out/s34_bench.err; echo bench_rc=$?
python -c "
import json;d=json.loads(open('gpurun_out/s34_bench.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['parity']['bitwise_equal'], d['clocks'])
for c in d.get('configs', []): print(c.get('config'), c.get('engine'), c.get('function'), c.get('dtype'), c.get('value'), c.get('ms'), c.get('reference_ms'), c.get('us_per_iteration'), c.get('kernel','')[:50])"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/s34_ref.json 2> gpurun_out/s34_ref.err; echo ref_rc=$?
tail -c 600 gpurun_out/s34_ref.json
