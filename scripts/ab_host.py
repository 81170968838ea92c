"""Same-box interleaved A/B of one library option on the host entry
(tbf_bilateral_trig_host: pinned input, H2D, filter, D2H, counters), one plan
per value (development aid).
usage: ab_host.py CONFIG OPTION VALUE_A VALUE_B [ROUNDS]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1105_4204_b200 as tb
from paper_1105_4204_b200 import _native, workloads

cfg = workloads.CONFIGS[int(sys.argv[1])]
opt, va, vb = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
rounds = int(sys.argv[5]) if len(sys.argv) > 5 else 6
lib = _native.load()
host = workloads.make_input(cfg, frames=min(cfg.frames, 8))
pin = torch.from_numpy(host).pin_memory()
out = torch.empty_like(pin).pin_memory()
k = tb.make_trig_kernel(cfg.sigma_r, cfg.T)
spec = tb.SpatialSpec.gaussian_recursive(cfg.sigma_s)
plans = {}
for v in (va, vb):
    lib.tbf_set_option(opt, v)
    plans[v] = tb.TrigFilter(tuple(pin.shape), spec, k)
res = {va: [], vb: []}
for r in range(rounds):
    for v in (va, vb):
        lib.tbf_set_option(opt, v)
        plans[v].run_host(pin, out)
        plans[v].read_counters()
        for _ in range(4):
            torch.cuda.synchronize()
            t = time.perf_counter()
            plans[v].run_host(pin, out)
            plans[v].read_counters()
            res[v].append(time.perf_counter() - t)
for v in (va, vb):
    print(f"{cfg.name} host entry, option {opt}={v}: median {1e3 * np.median(res[v]):.4f} ms  "
          f"min {1e3 * min(res[v]):.4f}", flush=True)
