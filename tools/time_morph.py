"""Time one morph op with CUDA events over rotating buffers (> L2), launched from a CUDA graph of
NB ops so host launch overhead is out of the picture:
python tools/time_morph.py W H wx wy op elem [--nograph]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2002_09474_b200 as pkg
W, H, wx, wy, op, elem = (int(v) for v in sys.argv[1:7])
use_graph = "--nograph" not in sys.argv
dt = torch.uint8 if elem == 1 else torch.uint16
nbytes = W * H * elem
NB = max(2, min(64, int(2 * 512e6 // (2 * nbytes)))) if nbytes < 256e6 else 2
srcs = [torch.empty((H, W), dtype=dt, device="cuda") for _ in range(NB)]
for s in srcs: pkg.generate_device(s, 2)
dsts = [torch.empty_like(s) for s in srcs]
for i in range(NB): pkg.morph_device(srcs[i], dsts[i], wx, wy, op)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
if use_graph:
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.graph(g, stream=s):
        for i in range(NB): pkg.morph_device(srcs[i], dsts[i], wx, wy, op)
    g.replay(); torch.cuda.synchronize()
    reps = max(1, 40 // NB)
    ev[0].record()
    for _ in range(reps): g.replay()
    ev[1].record(); torch.cuda.synchronize()
    n = reps * NB
else:
    n = 40
    ev[0].record()
    for i in range(n): pkg.morph_device(srcs[i % NB], dsts[i % NB], wx, wy, op)
    ev[1].record(); torch.cuda.synchronize()
us = ev[0].elapsed_time(ev[1]) / n * 1e3
print(f"{W}x{H} w={wx}x{wy} op={op} elem={elem} {'graph' if use_graph else 'eager'}: {us:.2f} us  {2*nbytes/us/1e3:.0f} GB/s  "
      f"{2*nbytes/us/1e3/6521.1*100:.1f}%  {pkg.plan_name(elem, W, H, wx, wy, op)}")
