cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_lazy.py tests/test_bench_parity.py -q -x > gpurun_out/s7_lazy.log 2>&1; echo lazy_rc=$?
tail -5 gpurun_out/s7_lazy.log
python - <<'PY'
import ctypes as C, sys
sys.path.insert(0, '.')
from paper_2408_00018_b200 import _abi
lib = _abi.load_library()
for prec in (0, 1):
    out = (C.c_uint64 * 3)()
    lib.psa_device_metropolis_check(prec, 777, 1 << 32, out)
    print("metropolis_check prec", prec, list(out))
PY
timeout 600 python scripts/lazy_rates.py > gpurun_out/s7_rates_f32.jsonl 2>&1; echo rates=$?
timeout 600 python scripts/lazy_rates.py --n 500 > gpurun_out/s7_rates_n500.jsonl 2>&1; echo rates500=$?
timeout 600 python scripts/lazy_rates.py --precision f64 > gpurun_out/s7_rates_f64.jsonl 2>&1; echo rates64=$?
for f in gpurun_out/s7_rates*.jsonl; do echo $f; python -c "
import json,sys
for l in open('$f'):
    try: d=json.loads(l)
    except Exception: print(l[:200]); continue
    print(d['t0'], '%.3e'%d['lazy']['evals_per_s'], '%.2e'%d['lazy']['exact_settle_frac'], '%.3e'%d['fold']['evals_per_s'])
"; done
timeout 900 python bench.py --no-companion > gpurun_out/s7_bench.json 2> gpurun_out/s7_bench.err; echo bench_rc=$?
python -c "
import json;d=json.loads(open('gpurun_out/s7_bench.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['roofline']['kernel'], d['parity']['bitwise_equal'])
for c in d.get('configs', []): print(c.get('config'), c.get('engine'), c.get('function'), c.get('dtype'), c.get('value'), c.get('us_per_iteration'), c.get('kernel','')[:40])"
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/s7_pytest.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/s7_pytest.log
