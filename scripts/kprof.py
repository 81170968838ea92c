"""Per-kernel event times of one config through one library build, in its own
process (development aid).  usage: kprof.py CONFIG[,CONFIG..] [LIB] [CALLS]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1105_4204_b200 as tb
from paper_1105_4204_b200 import _native, workloads

lib = _native.load(sys.argv[2] if len(sys.argv) > 2 and sys.argv[2] != "-" else None)
calls = int(sys.argv[3]) if len(sys.argv) > 3 else 3
nk = lib.tbf_profile_kinds()
for opt in os.environ.get("TBF_OPTS", "").split(","):  # e.g. TBF_OPTS=14=0,15=1
    if opt:
        o, v = opt.split("=")
        lib.tbf_set_option(int(o), int(v))
flush = torch.empty(128 << 20, device="cuda")
for cid in [int(c) for c in sys.argv[1].split(",")]:
    cfg = workloads.CONFIGS[cid]
    f = torch.from_numpy(workloads.make_input(cfg, frames=cfg.frames)).cuda()
    bt = os.environ.get("TBF_BT")  # terms per batch (default: the engine's pick)
    plan = tb.TrigFilter(tuple(f.shape), tb.SpatialSpec.gaussian_recursive(cfg.sigma_s),
                         tb.make_trig_kernel(cfg.sigma_r, cfg.T), batch_terms=int(bt) if bt else None)
    out = torch.empty_like(f)
    plan(f, out)
    torch.cuda.synchronize()
    tot, per = [], {}
    for _ in range(calls):
        flush.zero_()
        lib.tbf_profile_enable(1)
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        plan(f, out)
        b.record()
        torch.cuda.synchronize()
        lib.tbf_profile_enable(0)
        ms = (ctypes.c_double * nk)()
        ln = (ctypes.c_longlong * nk)()
        lib.tbf_profile_collect(ms, ln, nk)
        tot.append(a.elapsed_time(b))
        for i in range(nk):
            if ln[i]:
                per.setdefault(lib.tbf_kernel_name(i).decode(), []).append(ms[i])
    print(f"{cfg.name} {os.path.basename(sys.argv[2]) if len(sys.argv) > 2 else 'default'} {os.environ.get('TBF_OPTS', '')} bt={plan.batch_terms}: "
          f"{np.median(tot):.3f} ms  " + "  ".join(f"{k} {np.median(v):.3f}" for k, v in per.items()), flush=True)
    del plan, f, out
    torch.cuda.empty_cache()
