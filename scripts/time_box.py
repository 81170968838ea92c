"""Time the box spatial variant at config-2 scale (development aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1105_4204_b200 as tb
from paper_1105_4204_b200 import workloads
cfg = workloads.CONFIGS[2]
f = torch.from_numpy(workloads.make_input(cfg)).cuda()
k = tb.make_trig_kernel(cfg.sigma_r, cfg.T)
for r in (1, 8, 32):
    plan = tb.TrigFilter(tuple(f.shape), tb.SpatialSpec.box(r), k)
    out = plan(f); torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); plan(f, out); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    print(f"box r={r}: {np.median(ts):.3f} ms  ({f.numel()/np.median(ts)/1e3:.0f} Mpx/s)", flush=True)
