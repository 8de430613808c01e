"""Time one morph op with CUDA events over rotating buffers (> L2): python tools/time_morph.py W H wx wy op elem"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2002_09474_b200 as pkg
W, H, wx, wy, op, elem = (int(v) for v in sys.argv[1:7])
dt = torch.uint8 if elem == 1 else torch.uint16
nbytes = W * H * elem
NB = max(2, int(2 * 512e6 // (2 * nbytes)) if nbytes < 256e6 else 2)
NB = min(NB, 64)
srcs = [torch.empty((H, W), dtype=dt, device="cuda") for _ in range(NB)]
for s in srcs: pkg.generate_device(s, 2)
dsts = [torch.empty_like(s) for s in srcs]
for i in range(3): pkg.morph_device(srcs[i % NB], dsts[i % NB], wx, wy, op)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
reps = 40
ev[0].record()
for i in range(reps): pkg.morph_device(srcs[i % NB], dsts[i % NB], wx, wy, op)
ev[1].record(); torch.cuda.synchronize()
us = ev[0].elapsed_time(ev[1]) / reps * 1e3
print(f"{W}x{H} w={wx}x{wy} elem={elem} rh={os.environ.get('RMGPU_STREAM_RH','auto')}: {us:.2f} us  {2*nbytes/us/1e3:.0f} GB/s  {2*nbytes/us/1e3/6521.1*100:.1f}%  {pkg.plan_name(elem, W, H, wx, wy, op)}")
