"""Launch a few morph ops for profiling under ncu: python tools/prof_morph.py W H wx wy [op] [elem] [reps]"""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2002_09474_b200 as pkg

W, H, wx, wy = (int(v) for v in sys.argv[1:5])
op = int(sys.argv[5]) if len(sys.argv) > 5 else 0
elem = int(sys.argv[6]) if len(sys.argv) > 6 else 1
reps = int(sys.argv[7]) if len(sys.argv) > 7 else 3
dt = torch.uint8 if elem == 1 else torch.uint16
src = torch.empty((H, W), dtype=dt, device="cuda")
pkg.generate_device(src, 2)
dst = torch.empty_like(src)
for _ in range(reps):
    pkg.morph_device(src, dst, wx, wy, op)
torch.cuda.synchronize()
print("ok", pkg.plan_name(elem, W, H, wx, wy, op))
