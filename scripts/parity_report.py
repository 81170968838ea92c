"""Max abs error of the device filter against the committed reference goldens
(configs 1-5) and the oracle on large-sigma shapes, for one or more library
builds (development aid).  usage: parity_report.py [LIB ...]"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import paper_1105_4204_b200 as tb
from oracle import trigbf_oracle as orc
from paper_1105_4204_b200 import _native, engines, workloads

libs = sys.argv[1:] or [_native.LIB_PATH]
for p in libs:
    lib = ctypes.CDLL(os.path.abspath(p))
    _native._declare(lib)
    _native._lib = lib
    engines.clear_plans()
    res = []
    for cid in (1, 2, 3, 4, 5):
        g = np.load(os.path.join(ROOT, "tests", "golden", f"config_{cid}.npz"))
        cfg = workloads.CONFIGS[cid]
        k = tb.make_trig_kernel(cfg.sigma_r, cfg.T)
        spec = tb.SpatialSpec.gaussian_recursive(cfg.sigma_s)
        worst = 0.0
        for fi in sorted(set(g["frame"].tolist())):
            f = torch.from_numpy(workloads.frame(cfg, fi)).cuda()
            out = tb.bilateral_trig(f, spec, k)
            sel = g["frame"] == fi
            got = out[torch.from_numpy(g["y"][sel]).cuda(), torch.from_numpy(g["x"][sel]).cuda()]
            worst = max(worst, float(np.max(np.abs(got.double().cpu().numpy() - g["value"][sel]))))
            del out, f
        engines.clear_plans()
        res.append(f"cfg{cid} {worst:.3g}")
    for (h, w, s, sr) in [(300, 200, 100.0, 80.0), (540, 720, 100.0, 80.0), (64, 900, 300.0, 20.0),
                          (900, 64, 60.0, 30.0), (130, 70, 16.0, 10.0), (50, 300, 4.0, 40.0)]:
        f = np.random.default_rng(h + w).uniform(0, 255, (h, w)).astype(np.float32)
        got = tb.bilateral_trig(torch.from_numpy(f).cuda(), tb.SpatialSpec.gaussian_recursive(s),
                                tb.make_trig_kernel(sr, 255.0)).cpu().numpy()
        ref, _ = orc.bilateral_trig(f.astype(np.float64), "gauss-recursive", s, orc.make_trig_kernel(sr, 255.0))
        res.append(f"{h}x{w}/s{s:g}/r{sr:g} {np.max(np.abs(got - ref)):.3g}")
    print(os.path.basename(p) + ": " + "  ".join(res), flush=True)
