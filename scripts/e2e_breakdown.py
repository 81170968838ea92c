"""Where the single-image e2e time goes (development aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1105_4204_b200 as tb
from paper_1105_4204_b200 import workloads

cfg = workloads.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 2]
host = workloads.make_input(cfg, frames=1)[0]
pin = torch.from_numpy(host).pin_memory()
k = tb.make_trig_kernel(cfg.sigma_r, cfg.T)
spec = tb.SpatialSpec.gaussian_recursive(cfg.sigma_s)
dev = torch.device("cuda")


def timeit(fn, n=10, w=3):
    ts = []
    for i in range(w + n):
        torch.cuda.synchronize()
        t = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t)
    ts = ts[w:]
    return 1e3 * float(np.median(ts)), 1e3 * min(ts)


d_in = pin.to(dev)
out_pin = torch.empty_like(pin).pin_memory()
plan = tb.get_plan((1, *host.shape), spec, k, device=dev)
d_out = plan(d_in)
print("h2d        %.3f / %.3f ms" % timeit(lambda: d_in.copy_(pin, non_blocking=True)))
print("d2h        %.3f / %.3f ms" % timeit(lambda: out_pin.copy_(d_out.reshape(pin.shape), non_blocking=True)))
print("plan(f)    %.3f / %.3f ms" % timeit(lambda: plan(d_in, d_out)))
print("plan+ctr   %.3f / %.3f ms" % timeit(lambda: (plan(d_in, d_out), plan.read_counters())))
print("api pinned %.3f / %.3f ms" % timeit(lambda: tb.bilateral_trig(pin, spec, k)))
print("api numpy  %.3f / %.3f ms" % timeit(lambda: tb.bilateral_trig(host, spec, k)))
