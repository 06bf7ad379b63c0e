cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 python scripts/sanitize_runs.py > gpurun_out/s28_sanitizer_racecheck.log 2>&1; echo racecheck=$?
tail -3 gpurun_out/s28_sanitizer_racecheck.log
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/s28_pytest.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/s28_pytest.log
python - <<'PY'
import sys, time, json
sys.path.insert(0, '.')
import paper_2408_00018_b200 as psa
f = psa.registry_get("F0_a").with_dim(10)
cfg = psa.EngineConfig(n_chains=1, schedule=psa.AnnealSchedule(1000.0, 0.01, 0.99, 100), precision=psa.Precision.f32)
psa.run_sequential(f, cfg)
for _ in range(3):
    t0 = time.perf_counter(); r = psa.run_sequential(f, cfg); dt = time.perf_counter() - t0
    print(json.dumps({"v0_ms_e2e": dt * 1e3, "evals": r.evaluations, "best_f": r.best_f}))
PY
