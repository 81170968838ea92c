"""e2e of the frame-streamed path (config 4) vs sub-batch size (development aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1105_4204_b200 as tb
from paper_1105_4204_b200 import workloads
from paper_1105_4204_b200.engines import _bilateral_trig_streamed

cfg = workloads.CONFIGS[4]
host = workloads.make_input(cfg)
pin = torch.from_numpy(host).pin_memory()
k = tb.make_trig_kernel(cfg.sigma_r, cfg.T)
spec = tb.SpatialSpec.gaussian_recursive(cfg.sigma_s)
for rep in range(2):
    for sub, edges in ((8, False), (8, True), (6, True), (10, True)):
        for _ in range(2):
            _bilateral_trig_streamed(pin, spec, k, None, sub=sub, edges=edges)
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            t = time.perf_counter()
            _bilateral_trig_streamed(pin, spec, k, None, sub=sub, edges=edges)
            ts.append(time.perf_counter() - t)
        ms = 1e3 * float(np.median(ts))
        print(f"sub {sub:2d} edges {edges}: {ms:.2f} ms  {cfg.pixels / ms / 1e3:.0f} Mpx/s", flush=True)
