"""Time pass-1 y-chunk splits (TBF_P1_YSPLIT row counts) or pass-2 x-chunk
splits (TBF_P2_XSPLIT tile counts) on a config, interleaved over rounds with
one plan per variant; reports the step time, the pass time and the output
change against the first variant (development aid).
usage: sweep_ysplit.py CONFIG 'split:order;split:order;...' [x] [ROUNDS]
  split '' = automatic; order = pass-1 block order (-1 auto), or with x the
  pass-2 order for the explicit split (TBF_P2_XORDER, '' = default)"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1105_4204_b200 as tb
from paper_1105_4204_b200 import _native, workloads

cfg = workloads.CONFIGS[int(sys.argv[1])]
variants = [v.split(":") for v in sys.argv[2].split(";")]
xmode = len(sys.argv) > 3 and sys.argv[3] == "x"
rounds = int(sys.argv[4]) if len(sys.argv) > 4 else 4
lib = _native.load()
f = torch.from_numpy(workloads.make_input(cfg, frames=min(cfg.frames, 8))).cuda()
k = tb.make_trig_kernel(cfg.sigma_r, cfg.T)
spec = tb.SpatialSpec.gaussian_recursive(cfg.sigma_s)
flush = torch.empty(128 << 20, device="cuda")
KK = 4 if xmode else 2  # kernel timed: pass2 or pass1


def setv(split, order):
    os.environ["TBF_P2_XSPLIT" if xmode else "TBF_P1_YSPLIT"] = split
    if xmode:
        os.environ["TBF_P2_XORDER"] = order
    else:
        lib.tbf_set_option(10, int(order))


plans, outs = [], []
for split, order in variants:
    setv(split, order)
    plans.append(tb.TrigFilter(tuple(f.shape), spec, k))
    outs.append(torch.empty_like(f))
ts = [[] for _ in variants]
kt = [[] for _ in variants]
for r in range(rounds):
    for j, (split, order) in enumerate(variants):
        setv(split, order)
        plans[j](f, outs[j])
        for _ in range(3):
            flush.zero_()
            lib.tbf_profile_enable(1)
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            plans[j](f, outs[j])
            b.record()
            torch.cuda.synchronize()
            ms = (ctypes.c_double * 16)()
            cnt = (ctypes.c_longlong * 16)()
            lib.tbf_profile_collect(ms, cnt, 16)
            lib.tbf_profile_enable(0)
            ts[j].append(a.elapsed_time(b))
            kt[j].append(ms[KK])
for j, (split, order) in enumerate(variants):
    d = (outs[j] - outs[0]).abs().max().item()
    print(f"{cfg.name} split={split or 'auto':16s} order={order or '-':2s} step {np.median(ts[j]):.4f} ms  "
          f"{'pass2' if xmode else 'pass1'} {np.median(kt[j]):.4f} ms  max|diff| vs first {d:.2e}", flush=True)
