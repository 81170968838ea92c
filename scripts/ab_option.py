"""Same-box interleaved A/B of one library option on a config (development aid).
usage: ab_option.py CONFIG OPTION VALUE_A VALUE_B [ROUNDS]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1105_4204_b200 as tb
from paper_1105_4204_b200 import _native, workloads

cfg = workloads.CONFIGS[int(sys.argv[1])]
opt, va, vb = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
rounds = int(sys.argv[5]) if len(sys.argv) > 5 else 6
lib = _native.load()
f = torch.from_numpy(workloads.make_input(cfg, frames=min(cfg.frames, 8))).cuda()
k = tb.make_trig_kernel(cfg.sigma_r, cfg.T)
spec = tb.SpatialSpec.gaussian_recursive(cfg.sigma_s)
flush = torch.empty(128 << 20, device="cuda")
# one plan per value: an option may change the layout and so the workspace size
plans = {}
for v in (va, vb):
    lib.tbf_set_option(opt, v)
    plans[v] = tb.TrigFilter(tuple(f.shape), spec, k)
out = torch.empty_like(f)
res = {va: [], vb: []}
for r in range(rounds):
    for v in (va, vb):
        lib.tbf_set_option(opt, v)
        plan = plans[v]
        plan(f, out)
        for _ in range(5):
            flush.zero_()
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(); plan(f, out); b.record(); torch.cuda.synchronize()
            res[v].append(a.elapsed_time(b))
for v in (va, vb):
    print(f"{cfg.name} option {opt}={v}: median {np.median(res[v]):.4f} ms  mean {np.mean(res[v]):.4f}", flush=True)
