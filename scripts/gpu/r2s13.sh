cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:v2_lazy -c 1 -o gpurun_out/s13_lazy_hiT -f python scripts/profile_engine.py --tmin 905 --launches 1 > gpurun_out/s13_ncu1.log 2>&1; echo ncu1=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:v2_lazy -c 1 -o gpurun_out/s13_lazy_loT -f python scripts/profile_engine.py --t0 0.1 --tmin 0.0905 --launches 1 > gpurun_out/s13_ncu2.log 2>&1; echo ncu2=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s13_launches.csv python bench.py --steps 2 --warmup 1 --no-configs --no-cpu-baseline --no-companion > gpurun_out/s13_b_ncu.log 2>&1; echo ncul=$?
timeout 900 python bench.py > gpurun_out/s13_bench.json 2> gpurun_out/s13_bench.err; echo bench_rc=$?
python -c "
import json;d=json.loads(open('gpurun_out/s13_bench.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'], d['parity']['bitwise_equal'])
for c in d.get('configs', []): print(c.get('config'), c.get('engine'), c.get('function'), c.get('dtype'), c.get('value'), c.get('us_per_iteration'), c.get('kernel','')[:40], (c.get('roofline') or {}).get('frac'))"
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/s13_pytest.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/s13_pytest.log
