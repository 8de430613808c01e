"""One morph call (for compute-sanitizer / debugging): python tools/one_morph.py W H wx wy op elem"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2002_09474_b200 as pkg
W, H, wx, wy, op, elem = (int(v) for v in sys.argv[1:7])
dt = torch.uint8 if elem == 1 else torch.uint16
src = torch.empty((H, W), dtype=dt, device="cuda"); pkg.generate_device(src, 2)
dst = torch.empty_like(src)
pkg.morph_device(src, dst, wx, wy, op)
torch.cuda.synchronize()
print("ok", pkg.plan_name(elem, W, H, wx, wy, op))
