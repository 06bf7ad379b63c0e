import time, sys
sys.path.insert(0,'.')
import paper_2408_00018_b200 as psa
f = psa.registry_get("F0_a").with_dim(100)
for chains in (1024, 1<<20):
    cfg = psa.EngineConfig(n_chains=chains, schedule=psa.AnnealSchedule(1000.0, 999.0, 0.99, 1), precision=psa.Precision.f32)
    psa.run_synchronous(f, cfg)
    ts=[]
    for i in range(5):
        t0=time.perf_counter(); psa.run_synchronous(f, cfg); ts.append(time.perf_counter()-t0)
    print(chains, 'run_synchronous (1 level, N=1) ms:', [round(t*1e3,2) for t in ts])
