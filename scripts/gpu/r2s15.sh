cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_lazy.py -q -x > gpurun_out/s15_lazy.log 2>&1; echo lazy_rc=$?
tail -3 gpurun_out/s15_lazy.log
for a in "--n 100" "--n 500" "--n 500 --precision f64"; do
  timeout 600 python scripts/lazy_rates.py $a > gpurun_out/s15_rates.jsonl 2>&1
  echo "$a"; python -c "
import json
for l in open('gpurun_out/s15_rates.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l[:200]); continue
    print(d['t0'], '%.3e'%d['lazy']['evals_per_s'], '%.2e'%d['lazy']['exact_settle_frac'], d['lazy']['kernel'], '%.3e'%d['fold']['evals_per_s'])
"
done
