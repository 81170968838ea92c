"""Time tbf_bilateral_trig_host over strip/band counts (development aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1105_4204_b200 as tb
from paper_1105_4204_b200 import _native, workloads

cfg = workloads.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 2]
host = workloads.make_input(cfg, frames=1)
pin = torch.from_numpy(host).pin_memory()
out = torch.empty_like(pin).pin_memory()
k = tb.make_trig_kernel(cfg.sigma_r, cfg.T)
spec = tb.SpatialSpec.gaussian_recursive(cfg.sigma_s)
plan = tb.get_plan(tuple(pin.shape), spec, k)
lib = _native.load()
S = [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "0,2,3,4,6,8").split(",")]
Bn = [int(v) for v in (sys.argv[3] if len(sys.argv) > 3 else "0,2,3,4,6,8").split(",")]
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 13
for strips in S:
    for bands in Bn:
        lib.tbf_set_option(_native.TBF_OPT_HOST_STRIPS, strips)
        lib.tbf_set_option(_native.TBF_OPT_HOST_BANDS, bands)
        ts = []
        for i in range(reps):
            torch.cuda.synchronize()
            t = time.perf_counter()
            plan.run_host(pin, out)
            plan.read_counters()
            ts.append(time.perf_counter() - t)
        print(f"{cfg.name} strips {strips:2d} bands {bands:2d}  median {1e3*np.median(ts[2:]):.3f} ms  min {1e3*min(ts[2:]):.3f}", flush=True)
