cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_lazy.py tests/test_bench_parity.py -q -x > gpurun_out/s10_lazy.log 2>&1; echo lazy_rc=$?
tail -3 gpurun_out/s10_lazy.log
for m in "" lazy1; do
  PSA_V2_MODE=$m timeout 600 python scripts/lazy_rates.py > gpurun_out/s10_rates_$m.jsonl 2>&1
  echo mode=$m; python -c "
import json
for l in open('gpurun_out/s10_rates_$m.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l[:200]); continue
    print(d['t0'], '%.3e'%d['lazy']['evals_per_s'], '%.2e'%d['lazy']['exact_settle_frac'], d['lazy']['kernel'])
"
done
