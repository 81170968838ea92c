"""Timeline of one tbf_bilateral_trig_host call (development aid)."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1105_4204_b200 as tb
from paper_1105_4204_b200 import _native, workloads

cfg = workloads.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 2]
host = workloads.make_input(cfg, frames=1)
pin = torch.from_numpy(host).pin_memory()
out = torch.empty_like(pin).pin_memory()
k = tb.make_trig_kernel(cfg.sigma_r, cfg.T)
spec = tb.SpatialSpec.gaussian_recursive(cfg.sigma_s)
plan = tb.get_plan(tuple(pin.shape), spec, k)
lib = _native.load()
for _ in range(5):
    plan.run_host(pin, out); plan.read_counters()
lib.tbf_profile_enable(1)
cap = 256
st, du, kd = (ctypes.c_double * cap)(), (ctypes.c_double * cap)(), (ctypes.c_int32 * cap)()
for rep in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    plan.run_host(pin, out); plan.read_counters()
    wall = 1e3 * (time.perf_counter() - t)
    n = lib.tbf_profile_timeline(st, du, kd, cap)
    print(f"call {rep}: wall {wall:.3f} ms, {n} records")
    if rep == 2:
        for i in range(n):
            print(f"  {lib.tbf_kernel_name(kd[i]).decode():12s} start {st[i]:9.3f}  dur {du[i]:8.3f}  end {st[i] + du[i]:9.3f}")
        span = {}
        for i in range(n):
            nm = lib.tbf_kernel_name(kd[i]).decode()
            a, b, d = span.get(nm, (1e30, -1e30, 0.0))
            span[nm] = (min(a, st[i]), max(b, st[i] + du[i]), d + du[i])
        for nm, (a, b, d) in span.items():
            print(f"  summary {nm:12s} first start {a:9.3f}  last end {b:9.3f}  busy {d:9.3f} ms")
lib.tbf_profile_enable(0)
