"""Same-box interleaved A/B of two library builds on BASELINE configs, with a
bit-exactness check of their outputs (development aid).
usage: ab_libs.py LIB_A LIB_B [CONFIGS (e.g. 2,3,4)] [ROUNDS]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1105_4204_b200 as tb
from paper_1105_4204_b200 import _native, workloads

libs = sys.argv[1:3]
cfgs = [int(c) for c in (sys.argv[3] if len(sys.argv) > 3 else "2").split(",")]
rounds = int(sys.argv[4]) if len(sys.argv) > 4 else 6
handles = []
for p in libs:
    lib = ctypes.CDLL(os.path.abspath(p))

    class _Tolerant:  # an older build may lack the newest entry points
        def __getattr__(self, name):
            try:
                return getattr(lib, name)
            except AttributeError:
                return type("Missing", (), {})()

    _native._declare(_Tolerant())
    handles.append(lib)
flush = torch.empty(128 << 20, device="cuda")
for ci in cfgs:
    cfg = workloads.CONFIGS[ci]
    f = torch.from_numpy(workloads.make_input(cfg, frames=min(cfg.frames, 8))).cuda()
    k = tb.make_trig_kernel(cfg.sigma_r, cfg.T)
    spec = tb.SpatialSpec.gaussian_recursive(cfg.sigma_s)
    plans, outs = [], []
    for lib in handles:
        _native._lib = lib
        plans.append(tb.TrigFilter(tuple(f.shape), spec, k))
        outs.append(torch.empty_like(f))
    res = [[] for _ in handles]
    for r in range(rounds):
        for j, (plan, out) in enumerate(zip(plans, outs)):
            plan(f, out)
            for _ in range(3):
                flush.zero_()
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record()
                plan(f, out)
                b.record()
                torch.cuda.synchronize()
                res[j].append(a.elapsed_time(b))
    diff = (outs[0] - outs[1]).abs().max().item()
    same = torch.equal(outs[0], outs[1])
    line = f"{cfg.name}: " + "  ".join(
        f"{os.path.basename(libs[j])} median {np.median(res[j]):.4f} ms" for j in range(len(handles)))
    ratio = np.median(res[0]) / np.median(res[1])
    print(f"{line}  A/B {ratio:.4f}  bit-identical {same} (max diff {diff:.3g})", flush=True)
    del plans, outs
    torch.cuda.empty_cache()
