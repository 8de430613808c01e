"""Practical floor for one 1R+1W pass over an image: device-to-device copy of the same bytes, timed
like tools/time_morph.py (CUDA graph over rotating buffers). python tools/copy_floor.py W H elem"""
import sys
import torch
W, H, elem = (int(v) for v in sys.argv[1:4])
dt = torch.uint8 if elem == 1 else torch.uint16
nbytes = W * H * elem
NB = max(2, min(64, int(2 * 512e6 // (2 * nbytes)))) if nbytes < 256e6 else 2
srcs = [torch.empty((H, W), dtype=dt, device="cuda") for _ in range(NB)]
dsts = [torch.empty_like(s) for s in srcs]
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
with torch.cuda.graph(g, stream=s):
    for i in range(NB):
        dsts[i].copy_(srcs[i])
g.replay(); torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
reps = max(1, 40 // NB)
ev[0].record()
for _ in range(reps):
    g.replay()
ev[1].record(); torch.cuda.synchronize()
us = ev[0].elapsed_time(ev[1]) / (reps * NB) * 1e3
print(f"copy {W}x{H} elem={elem}: {us:.2f} us  {2*nbytes/us/1e3:.0f} GB/s  {2*nbytes/us/1e3/6521.1*100:.1f}%")
