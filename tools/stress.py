"""Repeat a morph op many times and check every result against the first (race detector)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2002_09474_b200 as pkg
W, H, wx, wy = (int(v) for v in sys.argv[1:5])
op = int(sys.argv[5]); elem = int(sys.argv[6]); reps = int(sys.argv[7])
dt = torch.uint8 if elem == 1 else torch.uint16
src = torch.empty((H, W), dtype=dt, device="cuda")
pkg.generate_device(src, 2)
ref = torch.empty_like(src)
pkg.morph_device(src, ref, wx, wy, op)
torch.cuda.synchronize()
bad = 0
out = torch.empty_like(src)
for i in range(reps):
    out.zero_() if elem == 1 else out.view(torch.uint8).zero_()
    pkg.morph_device(src, out, wx, wy, op)
    if i % 50 == 0 or i == reps - 1:
        torch.cuda.synchronize()
    if not torch.equal(out.view(torch.uint8), ref.view(torch.uint8)):
        bad += 1
torch.cuda.synchronize()
print("stress", sys.argv[1:], "mismatches", bad, "of", reps, pkg.plan_name(elem, W, H, wx, wy, op))
