cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_lazy.py -q -x -k "v0 or v1" > gpurun_out/s39_v0tests.log 2>&1; echo v0tests=$?; tail -2 gpurun_out/s39_v0tests.log
python - <<'PY'
import sys, time, json
sys.path.insert(0, '.')
import torch
import paper_2408_00018_b200 as psa
f = psa.registry_get("F0_a").with_dim(10)
for prec in (psa.Precision.f32, psa.Precision.f64):
    cfg = psa.EngineConfig(n_chains=1, schedule=psa.AnnealSchedule(1000.0, 0.01, 0.99, 100), precision=prec)
    with psa.Plan(f, cfg, engine=1) as p:
        s = torch.cuda.current_stream()
        p.launch(s.cuda_stream); p.fetch(s.cuda_stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s); p.launch(s.cuda_stream); e1.record(s); r = p.fetch(s.cuda_stream)
        print(json.dumps({"prec": prec.name, "v0_device_ms": e0.elapsed_time(e1), "best_f": r.best_f, "settles": p.exact_settles()}))
PY
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/s39_pytest.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/s39_pytest.log
timeout 900 python bench.py > gpurun_out/s39_bench.json 2> gpurun_out/s39_bench.err; echo bench_rc=$?
python -c "
import json;d=json.loads(open('gpurun_out/s39_bench.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['parity']['bitwise_equal'], d['clocks'])
for c in d.get('configs', []): print(c.get('config'), c.get('engine'), c.get('function'), c.get('dtype'), c.get('value'), c.get('ms'), c.get('reference_ms'), c.get('us_per_iteration'), c.get('kernel','')[:50])"
