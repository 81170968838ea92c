"""Run the device filter on a BASELINE config K times (profiling target).
usage: run_cfg.py CONFIG [CALLS] [FRAMES]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1105_4204_b200 as tb
from paper_1105_4204_b200 import workloads

cid = int(sys.argv[1])
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 1
cfg = workloads.CONFIGS[cid]
frames = int(sys.argv[3]) if len(sys.argv) > 3 else cfg.frames
f = torch.from_numpy(workloads.make_input(cfg, frames=frames)).cuda()
plan = tb.TrigFilter(tuple(f.shape), tb.SpatialSpec.gaussian_recursive(cfg.sigma_s), tb.make_trig_kernel(cfg.sigma_r, cfg.T))
out = torch.empty_like(f)
for _ in range(calls):
    plan(f, out)
torch.cuda.synchronize()
print("ok", cfg.name, float(out.mean()))
