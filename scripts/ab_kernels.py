"""Same-box interleaved A/B of several library builds with per-kernel times
(the library's event profiler) and the max difference to the first build.
usage: ab_kernels.py CONFIGS(e.g. 2,5) ROUNDS LIB [LIB ...]  (development aid)"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1105_4204_b200 as tb
from paper_1105_4204_b200 import _native, workloads

cfgs = [int(c) for c in sys.argv[1].split(",")]
rounds = int(sys.argv[2])
libs = sys.argv[3:]
handles = []
for p in libs:
    lib = ctypes.CDLL(os.path.abspath(p))
    _native._declare(lib)
    handles.append(lib)
flush = torch.empty(128 << 20, device="cuda")
for ci in cfgs:
    cfg = workloads.CONFIGS[ci]
    f = torch.from_numpy(workloads.make_input(cfg, frames=min(cfg.frames, 8))).cuda()
    k = tb.make_trig_kernel(cfg.sigma_r, cfg.T)
    spec = tb.SpatialSpec.gaussian_recursive(cfg.sigma_s)
    out = torch.empty_like(f)
    outs = []
    tot = [[] for _ in handles]
    per = [dict() for _ in handles]
    for r in range(rounds):
        for j, lib in enumerate(handles):
            _native._lib = lib
            plan = tb.TrigFilter(tuple(f.shape), spec, k)
            plan(f, out)
            torch.cuda.synchronize()
            if r == 0:
                outs.append(out.clone())
            for _ in range(2):
                flush.zero_()
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                with _native.KernelProfiler() as prof:
                    a.record()
                    plan(f, out)
                    b.record()
                    torch.cuda.synchronize()
                tot[j].append(a.elapsed_time(b))
                for name, (ms, n) in prof.result.items():
                    per[j].setdefault(name, []).append(ms)
            del plan
            torch.cuda.empty_cache()
    for j in range(len(handles)):
        d = float((outs[j] - outs[0]).abs().max())
        ks = "  ".join(f"{n} {np.median(v):.3f}" for n, v in per[j].items())
        print(f"cfg{ci} {os.path.basename(libs[j])}: total {np.median(tot[j]):.3f} ms | {ks} | maxdiff {d:.3g}",
              flush=True)
