"""Device time of one resident plan call across sigma_s (acceptance criterion 7:
time flat in sigma_s), with a per-kernel breakdown from torch.profiler.
Development aid: python scripts/sigma_sweep.py [H W] [sigma_r]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1105_4204_b200 as tb

H, W = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (2048, 2048)
sr = float(sys.argv[3]) if len(sys.argv) > 3 else 80.0
x = torch.from_numpy(np.random.default_rng(7).integers(0, 256, (H, W)).astype(np.float32)).cuda()
k = tb.make_trig_kernel(sr)
for ss in (3.0, 10.0, 30.0, 100.0, 300.0):
    plan = tb.TrigFilter((H, W), tb.SpatialSpec.gaussian_recursive(ss), k)
    out = plan(x)
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        plan(x, out)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA], acc_events=True) as prof:
        for _ in range(5):
            plan(x, out)
        torch.cuda.synchronize()
    per = {}
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            per[e.name] = per.get(e.name, 0.0) + e.device_time / 5e3
    def short(n):
        n = n.replace("void ", "").split("(")[0]
        return n.split("<")[0] + ("<" + n.split("<")[1].split(">")[0] + ">" if "<" in n else "")
    brk = ", ".join(f"{short(n)}={v:.3f}" for n, v in sorted(per.items(), key=lambda t: -t[1])[:6])
    print(f"{H}x{W} sigma_r={sr} N={k.N} sigma_s={ss}: {np.median(ts):.3f} ms | {brk}", flush=True)
