cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
./scripts/sort_probe > gpurun_out/s25_sort_probe.jsonl 2>&1; cat gpurun_out/s25_sort_probe.jsonl
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_bench_parity.py -q -x -k "nelder or hybrid or nm or c4" > gpurun_out/s25_nm_tests.log 2>&1; echo nmtests=$?
tail -2 gpurun_out/s25_nm_tests.log
timeout 1500 python scripts/nm_rate.py 1000000 3000000 > gpurun_out/s25_nm_rate.jsonl 2>&1; echo rc=$?
cat gpurun_out/s25_nm_rate.jsonl
for v in default p0add; do
  if [ $v = default ]; then L=paper_2408_00018_b200/libparsa_b200.so; else L=gpu_variants/$v/libparsa_b200.so; fi
  PSA_LIB_PATH=$L timeout 600 python scripts/lazy_rates.py > gpurun_out/s25_rates_$v.jsonl 2>&1
  echo $v; python -c "
import json
for l in open('gpurun_out/s25_rates_$v.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l[:200]); continue
    print(d['t0'], '%.3e'%d['lazy']['evals_per_s'], d['lazy']['kernel'])
"
done
