"""Time one config under several library options (development aid)."""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1105_4204_b200 as tb
from paper_1105_4204_b200 import _native, workloads

cfg = workloads.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 2]
lib = _native.load()
f = torch.from_numpy(workloads.make_input(cfg, frames=min(cfg.frames, 8))).cuda()
k = tb.make_trig_kernel(cfg.sigma_r, cfg.T)
spec = tb.SpatialSpec.gaussian_recursive(cfg.sigma_s)
flush = torch.empty(128 << 20, device="cuda")
variants = [("default", {}), ("p2c1", {3: 1}), ("p2c2", {3: 2}), ("p2c3", {3: 3}), ("p2c4", {3: 4}), ("yc2", {5: 2}), ("yc3", {5: 3}), ("yc4", {5: 4})]
if len(sys.argv) > 2:  # variants as JSON: [["name", {"option": value}], ...]
    variants = [(n, {int(o): v for o, v in d.items()}) for n, d in json.loads(sys.argv[2])]
for name, opts in variants:
    for o, v in {0: 0, 2: 3, 3: 0, 4: 3, 1: 2, 5: 0, 6: 1, 9: 0, 10: -1}.items():
        lib.tbf_set_option(o, v)
    for o, v in opts.items():
        lib.tbf_set_option(o, v)
    plan = tb.TrigFilter(tuple(f.shape), spec, k)
    out = plan(f); torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); plan(f, out); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    print(f"{cfg.name} {name:10s} median {np.median(ts):8.3f} ms  min {min(ts):8.3f}", flush=True)
    del plan; torch.cuda.empty_cache()
