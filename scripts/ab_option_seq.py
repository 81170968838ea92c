"""Same-box A/B of one library option with one plan alive at a time (so the
term-batch picker sees the same free memory for both values), per-kernel
times from the library's event profiler (development aid).
usage: ab_option_seq.py CONFIGS OPTION VALUE_A VALUE_B [ROUNDS]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1105_4204_b200 as tb
from paper_1105_4204_b200 import _native, engines, workloads

cfgs = [int(c) for c in sys.argv[1].split(",")]
opt, va, vb = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
rounds = int(sys.argv[5]) if len(sys.argv) > 5 else 3
lib = _native.load()
flush = torch.empty(128 << 20, device="cuda")
for ci in cfgs:
    cfg = workloads.CONFIGS[ci]
    f = torch.from_numpy(workloads.make_input(cfg, frames=min(cfg.frames, 8))).cuda()
    k = tb.make_trig_kernel(cfg.sigma_r, cfg.T)
    spec = tb.SpatialSpec.gaussian_recursive(cfg.sigma_s)
    res = {va: [], vb: []}
    per = {va: {}, vb: {}}
    outs = {}
    for r in range(rounds):
        for v in (va, vb):
            lib.tbf_set_option(opt, v)
            plan = tb.TrigFilter(tuple(f.shape), spec, k)
            out = plan(f)
            torch.cuda.synchronize()
            outs[v] = out
            for _ in range(3):
                flush.zero_()
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                with _native.KernelProfiler() as prof:
                    a.record()
                    plan(f, out)
                    b.record()
                    torch.cuda.synchronize()
                res[v].append(a.elapsed_time(b))
                for name, (ms, n) in prof.result.items():
                    per[v].setdefault(name, []).append(ms)
            del plan
            engines.clear_plans()
    d = float((outs[va] - outs[vb]).abs().max())
    for v in (va, vb):
        ks = "  ".join(f"{n} {np.median(x):.3f}" for n, x in per[v].items())
        print(f"cfg{ci} option {opt}={v}: total {np.median(res[v]):.3f} ms | {ks} | maxdiff {d:.3g}", flush=True)
lib.tbf_set_option(opt, va)
