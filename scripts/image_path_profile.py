"""Break down host overhead of bilateral_trig(Image) on a small image (development aid)."""
import cProfile, pstats, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1105_4204_b200 as tb
from paper_1105_4204_b200.cli import synthesize_noise

img = synthesize_noise()
spec = tb.SpatialSpec.gaussian_recursive(10.0)
for sr in (100.0, 20.0, 10.0):
    k = tb.make_trig_kernel(sr)
    for _ in range(3):
        tb.bilateral_trig(img, spec, k)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(20):
        tb.bilateral_trig(img, spec, k)
    print(f"sigma_r {sr}: {1e3 * (time.perf_counter() - t) / 20:.3f} ms/call", flush=True)
    plan = tb.get_plan((1, 540, 720), spec, k)
    f = torch.from_numpy(np.ascontiguousarray(img.samples[0], dtype=np.float32)).cuda()
    out = torch.empty_like(f)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(20):
        plan(f, out)
    torch.cuda.synchronize()
    print(f"   device plan(f): {1e3 * (time.perf_counter() - t) / 20:.3f} ms/call", flush=True)
k = tb.make_trig_kernel(100.0)
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    tb.bilateral_trig(img, spec, k)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
