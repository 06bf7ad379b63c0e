cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_lazy.py tests/test_gpu_parity.py tests/test_reference_suites.py -q -x > gpurun_out/s31_tests.log 2>&1; echo tests=$?
tail -5 gpurun_out/s31_tests.log
python - <<'PY'
import sys, time, json
sys.path.insert(0, '.')
import torch
import paper_2408_00018_b200 as psa
f = psa.registry_get("F0_a").with_dim(10)
cfg = psa.EngineConfig(n_chains=1, schedule=psa.AnnealSchedule(1000.0, 0.01, 0.99, 100), precision=psa.Precision.f32)
with psa.Plan(f, cfg, engine=1) as p:
    print(p.description)
    s = torch.cuda.current_stream()
    p.launch(s.cuda_stream); p.fetch(s.cuda_stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s); p.launch(s.cuda_stream); e1.record(s); r = p.fetch(s.cuda_stream)
    print(json.dumps({"v0_device_ms": e0.elapsed_time(e1), "best_f": r.best_f, "settles": p.exact_settles()}))
PY
