"""Per-iteration timeline of one CTA of the streaming kernel: python tools/trace_stream.py W H wx wy elem cta"""
import sys, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2002_09474_b200 as pkg
W, H, wx, wy, elem, cta = (int(v) for v in sys.argv[1:7])
dt = torch.uint8 if elem == 1 else torch.uint16
src = torch.empty((H, W), dtype=dt, device="cuda"); pkg.generate_device(src, 2)
dst = torch.empty_like(src)
for _ in range(2): pkg.morph_device(src, dst, wx, wy, 0)
tr = torch.zeros(1024, dtype=torch.int64, device="cuda")
pkg.lib().rmgpu_debug_trace(C.c_void_p(tr.data_ptr()), cta)
pkg.morph_device(src, dst, wx, wy, 0)
torch.cuda.synchronize()
pkg.lib().rmgpu_debug_trace(None, 0)
t = tr.cpu().numpy()
t0 = min(v for v in t if v > 0)
print(pkg.plan_name(elem, W, H, wx, wy, 0))
print("iter |  VW: start  issued  data   empty  done |  HW: start  full  hdone  stored  end")
for L in range(60):
    v = [t[L * 8 + k] for k in range(5)]
    h = [t[480 + L * 8 + k] for k in range(5)]
    if max(v + h) == 0:
        continue
    f = lambda x: f"{(x - t0):7d}" if x else "      -"
    print(f"{L:4d} | " + " ".join(f(x) for x in v) + " | " + " ".join(f(x) for x in h))
