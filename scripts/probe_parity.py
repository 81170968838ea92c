"""Quick GPU parity probe across shapes/params (development aid)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1105_4204_b200 as tb
from oracle import trigbf_oracle as orc

rng = np.random.default_rng(0)
cases = [((1,1),3,30),((1,5),2,30),((5,1),2,30),((7,3),3,60),((40,30),3,60),((64,64),2,80),
         ((100,37),5,25),((33,65),8,20),((96,80),3,30),((130,70),16,10),((50,300),4,40),((1,1),1,100),
         ((64,64),2,500)]
worst = 0
for (h,w), ss, sr in cases:
    f = rng.uniform(0,255,(h,w)).astype(np.float32)
    k = tb.make_trig_kernel(sr, 255.0)
    t=time.time()
    got = tb.bilateral_trig(torch.from_numpy(f).cuda(), tb.SpatialSpec.gaussian_recursive(ss), k).cpu().numpy()
    ref,_ = orc.bilateral_trig(f.astype(np.float64), 'gauss-recursive', ss, orc.make_trig_kernel(sr,255.0))
    e = np.abs(got-ref).max(); worst=max(worst,e)
    print('gauss', (h,w), ss, sr, 'N=%d'%k.N, 'err=%.3g'%e, flush=True)
for (h,w), r, sr in [((16,16),1,30),((64,64),3,60),((20,10),2,80),((5,4),7,50),((37,53),0,30)]:
    f = rng.uniform(0,255,(h,w)).astype(np.float32)
    k = tb.make_trig_kernel(sr, 255.0)
    got = tb.bilateral_trig(torch.from_numpy(f).cuda(), tb.SpatialSpec.box(r), k).cpu().numpy()
    ref,_ = orc.bilateral_trig(f.astype(np.float64), 'box', r, orc.make_trig_kernel(sr,255.0))
    e = np.abs(got-ref).max(); worst=max(worst,e)
    print('box', (h,w), r, sr, 'N=%d'%k.N, 'err=%.3g'%e, flush=True)
print('WORST', worst)
