cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/s27_pytest.log 2>&1; echo pytest_rc=$?
tail -4 gpurun_out/s27_pytest.log
timeout 900 python bench.py > gpurun_out/s27_bench.json 2> gpurun_out/s27_bench.err; echo bench_rc=$?
python -c "
import json;d=json.loads(open('gpurun_out/s27_bench.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['roofline']['kernel'][:60], d['roofline']['frac'], d['parity']['bitwise_equal'], d['clocks'])
for c in d.get('configs', []): print(c.get('config'), c.get('engine'), c.get('function'), c.get('dtype'), c.get('value'), c.get('ms'), c.get('reference_ms'), c.get('us_per_iteration'), c.get('kernel','')[:40], (c.get('roofline') or {}).get('frac'))"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:v2_lazy -c 1 -o gpurun_out/s27_lazy_hiT -f python scripts/profile_engine.py --tmin 905 --launches 1 > gpurun_out/s27_ncu1.log 2>&1; echo ncu1=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s27_launches.csv python bench.py --steps 2 --warmup 1 --no-configs --no-cpu-baseline --no-companion > gpurun_out/s27_b_ncu.log 2>&1; echo ncul=$?
for tool in racecheck synccheck memcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_runs.py > gpurun_out/s27_sanitizer_$tool.log 2>&1; echo $tool=$?
  tail -4 gpurun_out/s27_sanitizer_$tool.log
done
