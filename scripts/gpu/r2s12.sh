cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in default u2 u4; do
  if [ $v = default ]; then L=paper_2408_00018_b200/libparsa_b200.so; else L=gpu_variants/$v/libparsa_b200.so; fi
  PSA_LIB_PATH=$L timeout 600 python scripts/lazy_rates.py > gpurun_out/s12_rates_$v.jsonl 2>&1
  echo $v; python -c "
import json
for l in open('gpurun_out/s12_rates_$v.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l[:200]); continue
    print(d['t0'], '%.3e'%d['lazy']['evals_per_s'], '%.2e'%d['lazy']['exact_settle_frac'])
"
done
