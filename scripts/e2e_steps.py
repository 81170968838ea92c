"""Per-step times of bench.py's e2e leg (public bilateral_trig on a pinned host
tensor), plus the pinned copy bandwidth of this host (development aid).
usage: e2e_steps.py [CONFIG] [STEPS]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1105_4204_b200 as tb
from paper_1105_4204_b200 import workloads

cfg = workloads.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 2]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
host = workloads.make_input(cfg)
pin_in = torch.from_numpy(host).pin_memory()
spec = tb.SpatialSpec.gaussian_recursive(cfg.sigma_s)
kernel = tb.make_trig_kernel(cfg.sigma_r, cfg.T)
ts = []
for i in range(3 + steps):
    torch.cuda.synchronize()
    t = time.perf_counter()
    res = tb.bilateral_trig(pin_in, spec, kernel)
    ts.append(1e3 * (time.perf_counter() - t))
ts = ts[3:]
print(f"{cfg.name} e2e steps (ms): " + " ".join(f"{v:.3f}" for v in ts))
print(f"  mean {np.mean(ts):.3f}  median {np.median(ts):.3f}  min {min(ts):.3f}  max {max(ts):.3f}")
# pinned copy bandwidth, each direction alone and both at once
d = torch.empty_like(pin_in, device="cuda")
o = torch.empty_like(pin_in).pin_memory()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for name, fn in (("h2d", lambda: d.copy_(pin_in, non_blocking=True)),
                 ("d2h", lambda: o.copy_(d, non_blocking=True))):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 10
    print(f"  {name} {pin_in.numel() * 4 / dt / 1e9:.1f} GB/s ({1e3 * dt:.3f} ms for {pin_in.numel() * 4 >> 20} MiB)")
