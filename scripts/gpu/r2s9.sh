cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_lazy.py tests/test_bench_parity.py -q -x > gpurun_out/s9_lazy.log 2>&1; echo lazy_rc=$?
tail -3 gpurun_out/s9_lazy.log
for v in default coef; do
  if [ $v = default ]; then L=paper_2408_00018_b200/libparsa_b200.so; else L=gpu_variants/$v/libparsa_b200.so; fi
  PSA_LIB_PATH=$L timeout 600 python scripts/lazy_rates.py > gpurun_out/s9_rates_$v.jsonl 2>&1
  echo $v; python -c "
import json
for l in open('gpurun_out/s9_rates_$v.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l[:200]); continue
    print(d['t0'], '%.3e'%d['lazy']['evals_per_s'], '%.2e'%d['lazy']['exact_settle_frac'])
"
done
