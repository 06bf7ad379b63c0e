cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_lazy.py tests/test_bench_parity.py -q -x > gpurun_out/s6_lazy.log 2>&1; echo lazy_rc=$?
tail -5 gpurun_out/s6_lazy.log
timeout 600 python scripts/lazy_rates.py > gpurun_out/s6_rates_f32.jsonl 2>&1; echo rates=$?
PSA_LIB_PATH=gpu_variants/unroll2/libparsa_b200.so timeout 600 python scripts/lazy_rates.py > gpurun_out/s6_rates_f32_u2.jsonl 2>&1; echo rates=$?
timeout 600 python scripts/lazy_rates.py --n 500 > gpurun_out/s6_rates_n500.jsonl 2>&1; echo rates500=$?
timeout 600 python scripts/lazy_rates.py --precision f64 > gpurun_out/s6_rates_f64.jsonl 2>&1; echo rates64=$?
for f in gpurun_out/s6_rates*.jsonl; do echo $f; python -c "
import json,sys
for l in open('$f'):
    try: d=json.loads(l)
    except Exception: print(l[:200]); continue
    print(d['t0'], '%.3e'%d['lazy']['evals_per_s'], '%.2e'%d['lazy']['exact_settle_frac'], '%.3e'%d['fold']['evals_per_s'])
"; done
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/s6_pytest.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/s6_pytest.log
