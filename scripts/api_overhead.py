"""Where the public API's per-call overhead goes on a pinned host tensor
(development aid).  usage: api_overhead.py CONFIG"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1105_4204_b200 as tb
from paper_1105_4204_b200 import workloads

cfg = workloads.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 2]
host = workloads.make_input(cfg, frames=1)
pin = torch.from_numpy(host).pin_memory()
k = tb.make_trig_kernel(cfg.sigma_r, cfg.T)
spec = tb.SpatialSpec.gaussian_recursive(cfg.sigma_s)


def t(fn, n=20):
    ts = []
    for _ in range(n):
        torch.cuda.synchronize()
        a = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - a)
    return 1e3 * float(np.median(ts[3:]))


plan = tb.get_plan(tuple(pin.shape), spec, k)
out = torch.empty_like(pin).pin_memory()
print("run_host+counters  %.3f ms" % t(lambda: (plan.run_host(pin, out), plan.read_counters())))
print("run_host only      %.3f ms (+sync)" % t(lambda: (plan.run_host(pin, out), torch.cuda.synchronize())))
print("read_counters      %.3f ms" % t(lambda: plan.read_counters()))
print("empty pinned       %.3f ms" % t(lambda: torch.empty(tuple(pin.shape), dtype=torch.float32, pin_memory=True)))
print("get_plan           %.3f ms" % t(lambda: tb.get_plan(tuple(pin.shape), spec, k)))
print("is_pinned          %.3f ms" % t(lambda: pin.is_pinned()))
print("api pinned         %.3f ms" % t(lambda: tb.bilateral_trig(pin, spec, k)))
import cProfile, pstats
pr = cProfile.Profile()
pr.enable()
for _ in range(10):
    tb.bilateral_trig(pin, spec, k)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
