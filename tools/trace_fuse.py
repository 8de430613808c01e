"""Per-block timeline of one CTA of the fused kernel K4:
python tools/trace_fuse.py W H wx wy elem cta"""
import sys, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2002_09474_b200 as pkg
W, H, wx, wy, elem, cta = (int(v) for v in sys.argv[1:7])
dt = torch.uint8 if elem == 1 else torch.uint16
src = torch.empty((H, W), dtype=dt, device="cuda"); pkg.generate_device(src, 2)
dst = torch.empty_like(src)
for _ in range(2): pkg.morph_device(src, dst, wx, wy, 0)
torch.cuda.synchronize()
tr = torch.zeros(2048, dtype=torch.int64, device="cuda")
pkg.lib().rmgpu_debug_trace(C.c_void_p(tr.data_ptr()), cta)
pkg.morph_device(src, dst, wx, wy, 0)
torch.cuda.synchronize()
pkg.lib().rmgpu_debug_trace(None, 0)
t = tr.cpu().numpy()
nz = [v for v in t if v > 0]
t0 = min(nz)
print(pkg.plan_name(elem, W, H, wx, wy, 0), "span", max(nz) - t0, "cycles")
print("V blk | wait0  full  tempty  done")
for c in range(64):
    v = [t[c * 8 + k] for k in (0, 1, 2, 3)]
    if max(v) == 0:
        continue
    print(f"{c:5d} | " + " ".join(f"{(x - t0):6d}" if x else "     -" for x in v))
for w in range(4):
    print(f"H warp {w} | wait0 ready done")
    for g in range(64):
        v = [t[1024 + w * 256 + g * 4 + k] for k in range(3)]
        if max(v) == 0:
            continue
        print(f"   {g:3d} | " + " ".join(f"{(x - t0):6d}" if x else "     -" for x in v))
print("refill (H warp 0) | test  tested  slept  issued")
for n in range(12):
    v = [t[1024 + 200 + n * 4 + k] for k in range(4)]
    if max(v) == 0:
        continue
    print(f"   {n:3d} | " + " ".join(f"{(x - t0):6d}" if x else "     -" for x in v))
