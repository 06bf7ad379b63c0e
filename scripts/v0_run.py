import sys
sys.path.insert(0, '.')
import paper_2408_00018_b200 as psa
f = psa.registry_get("F0_a").with_dim(10)
cfg = psa.EngineConfig(n_chains=1, schedule=psa.AnnealSchedule(1000.0, 0.01, 0.99, 100), precision=psa.Precision.f32)
print(psa.run_sequential(f, cfg).best_f)
