cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_lazy.py -q -x > gpurun_out/s16_lazy.log 2>&1; echo lazy_rc=$?
tail -3 gpurun_out/s16_lazy.log
for a in "--n 500" ; do
  timeout 600 python scripts/lazy_rates.py $a > gpurun_out/s16_rates_n500.jsonl 2>&1
  echo "$a"; python -c "
import json
for l in open('gpurun_out/s16_rates_n500.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l[:200]); continue
    print(d['t0'], '%.3e'%d['lazy']['evals_per_s'], '%.2e'%d['lazy']['exact_settle_frac'], d['lazy']['kernel'], '%.3e'%d['fold']['evals_per_s'])
"
done
timeout 900 python bench.py --steps 3 > gpurun_out/s16_bench.json 2> gpurun_out/s16_bench.err; echo bench_rc=$?
python -c "
import json;d=json.loads(open('gpurun_out/s16_bench.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'], d['parity']['bitwise_equal'])
for c in d.get('configs', []): print(c.get('config'), c.get('engine'), c.get('function'), c.get('dtype'), c.get('value'), c.get('us_per_iteration'), c.get('kernel','')[:50], (c.get('roofline') or {}).get('frac'))"
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/s16_pytest.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/s16_pytest.log
