"""Break down the public-API e2e call on a pinned host tensor (bench.py's e2e
leg) into plan lookup, output allocation, the host entry and the finish
(development aid).  usage: e2e_overhead.py [CONFIG]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1105_4204_b200 as tb
from paper_1105_4204_b200 import engines, workloads

cfg = workloads.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 2]
host = workloads.make_input(cfg, frames=1)[0]
pin = torch.from_numpy(host).pin_memory()
k = tb.make_trig_kernel(cfg.sigma_r, cfg.T)
spec = tb.SpatialSpec.gaussian_recursive(cfg.sigma_s)
shape = (1, *pin.shape)


def timeit(fn, n=20):
    ts = []
    for _ in range(n):
        torch.cuda.synchronize()
        t = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t)
    return 1e3 * np.median(ts[3:])


plan = engines.get_plan(shape, spec, k)
out = torch.empty(pin.shape, dtype=torch.float32, pin_memory=True)
print(f"{cfg.name}")
print(f"  public bilateral_trig(pinned)        {timeit(lambda: tb.bilateral_trig(pin, spec, k)):.4f} ms")
print(f"  get_plan                             {timeit(lambda: engines.get_plan(shape, spec, k)):.4f} ms")
print(f"  torch.empty(pin_memory=True)         {timeit(lambda: torch.empty(pin.shape, dtype=torch.float32, pin_memory=True)):.4f} ms")
print(f"  run_host + read_counters             {timeit(lambda: (plan.run_host(pin, out), plan.read_counters())):.4f} ms")
print(f"  run_host only (then sync)            {timeit(lambda: (plan.run_host(pin, out), torch.cuda.synchronize())):.4f} ms")
