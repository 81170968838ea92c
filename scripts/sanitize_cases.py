"""Small device calls covering every kernel path, for compute-sanitizer
(memcheck / racecheck / synccheck, one tool per run): recursive Gaussian
(stripes, x hand-off across stripes, y-chunks, x-chunks), box, batched
frames, the host entry (strips, bands), row-band partials, the zero unit and
cluster options, the brute force.  usage: sanitize_cases.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1105_4204_b200 as tb
from paper_1105_4204_b200 import _native
from paper_1105_4204_b200.workloads import smooth_image

lib = _native.load()
rng = np.random.default_rng(0)
f = torch.from_numpy(smooth_image(260, 300, 6, seed=1)).cuda()
k = tb.make_trig_kernel(30.0)
out = tb.bilateral_trig(f, tb.SpatialSpec.gaussian_recursive(4.0), k)
out = tb.bilateral_trig(f, tb.SpatialSpec.box(3), tb.make_trig_kernel(40.0))
fb = torch.from_numpy(rng.uniform(0, 255, (3, 70, 90)).astype(np.float32)).cuda()
out = tb.bilateral_trig(fb, tb.SpatialSpec.gaussian_recursive(2.0), tb.make_trig_kernel(60.0))
host = rng.uniform(0, 255, (1, 300, 520)).astype(np.float32)
lib.tbf_set_option(_native.TBF_OPT_HOST_STRIPS, 2)
lib.tbf_set_option(_native.TBF_OPT_HOST_BANDS, 2)
res = tb.bilateral_trig(torch.from_numpy(host).pin_memory(), tb.SpatialSpec.gaussian_recursive(3.0), k)
lib.tbf_set_option(_native.TBF_OPT_HOST_STRIPS, 0)
lib.tbf_set_option(_native.TBF_OPT_HOST_BANDS, 0)
g = torch.from_numpy(host).cuda()
n = tb.kernels.term_pairs(k).count
nd = torch.zeros((2, *g.shape), device="cuda")
tb.TrigFilter(tuple(g.shape), tb.SpatialSpec.gaussian_recursive(3.0), k, term_range=(0, n // 2)).partial(g, nd[0], nd[1])
tb.TrigFilter(tuple(g.shape), tb.SpatialSpec.gaussian_recursive(3.0), k, term_range=(n // 2, n)).partial(
    g, nd[0], nd[1], accumulate=True, rows=(128, 300))
lib.tbf_set_option(_native.TBF_OPT_ZERO_UNIT, 1)
out = tb.TrigFilter(tuple(g.shape), tb.SpatialSpec.gaussian_recursive(3.0), k)(g)
lib.tbf_set_option(_native.TBF_OPT_ZERO_UNIT, 0)
lib.tbf_set_option(_native.TBF_OPT_P1_CLUSTER, 4)
out = tb.TrigFilter(tuple(g.shape), tb.SpatialSpec.gaussian_recursive(3.0), k)(g)
lib.tbf_set_option(_native.TBF_OPT_P1_CLUSTER, 1)
# several term batches (workspace num/den accumulation, x-chunks of a multi-batch launch)
out = tb.TrigFilter(tuple(g.shape), tb.SpatialSpec.gaussian_recursive(3.0), k, batch_terms=4)(g)
d = tb.bilateral_direct(rng.uniform(0, 255, (20, 23)), tb.SpatialSpec.box(2), k)
torch.cuda.synchronize()
print("sanitize cases done")
