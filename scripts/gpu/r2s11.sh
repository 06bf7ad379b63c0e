cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_lazy.py tests/test_bench_parity.py -q -x > gpurun_out/s11_lazy.log 2>&1; echo lazy_rc=$?
tail -3 gpurun_out/s11_lazy.log
timeout 600 python scripts/lazy_rates.py > gpurun_out/s11_rates.jsonl 2>&1
python -c "
import json
for l in open('gpurun_out/s11_rates.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l[:200]); continue
    print(d['t0'], '%.3e'%d['lazy']['evals_per_s'], '%.2e'%d['lazy']['exact_settle_frac'], d['lazy']['kernel'], '%.3e'%d['fold']['evals_per_s'])
"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:v2_lazy -c 1 -o gpurun_out/s11_lazy_hiT -f python scripts/profile_engine.py --tmin 905 --launches 1 > gpurun_out/s11_ncu1.log 2>&1; echo ncu1=$?
