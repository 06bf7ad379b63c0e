"""Compare the device-timed plan launch with the end-to-end C-ABI call on
the bench workload (C2), interleaved, to separate host overhead from clock
or thermal effects.  Prints one line per measurement."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2408_00018_b200 as psa  # noqa: E402

f = psa.registry_get("F0_a").with_dim(100)
cfg = psa.EngineConfig(n_chains=1 << 20, schedule=psa.AnnealSchedule(1000.0, 0.01, 0.99, 100),
                       precision=psa.Precision.f32)
s = torch.cuda.current_stream()
with psa.Plan(f, cfg) as p:
    p.launch(s.cuda_stream)
    p.fetch(s.cuda_stream)
    for i in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        p.launch(s.cuda_stream)
        e1.record(s)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        p.fetch(s.cuda_stream)
        print("plan  device ms", round(e0.elapsed_time(e1), 1), "fetch ms", round(1e3 * (time.perf_counter() - t0), 2))
        t0 = time.perf_counter()
        r = psa.run_synchronous(f, cfg)
        torch.cuda.synchronize()
        print("e2e   wall ms", round(1e3 * (time.perf_counter() - t0), 1), "reported wall_time_s", round(r.wall_time_s * 1e3, 1))
