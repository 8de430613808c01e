"""Compare the GPU result with the oracle for one case and print where they differ:
python tools/diffcase.py W H wx wy op elem [border bval]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2002_09474_b200 as pkg
import oracle
from tests.gpu_util import to_device, empty_device, to_host
W, H, wx, wy, op, elem = (int(v) for v in sys.argv[1:7])
border = int(sys.argv[7]) if len(sys.argv) > 7 else 0
bval = int(sys.argv[8]) if len(sys.argv) > 8 else 0
dt = np.uint8 if elem == 1 else np.uint16
R = oracle.restatement()
img = R.generate(W, H, 7, dtype=dt)
want = R.morph(img, wx, wy, op, border, bval)
src = to_device(img, 0); dst = empty_device(img.shape, dt, 0)
pkg.morph_device(src, dst, wx, wy, op, border, bval); torch.cuda.synchronize()
got = to_host(dst)
bad = np.argwhere(got != want)
print(pkg.plan_name(elem, W, H, wx, wy, op), "mismatches", len(bad), "of", got.size)
if len(bad):
    rows = np.unique(bad[:, 0]); cols = np.unique(bad[:, 1])
    print("rows", rows[:20], "... n", len(rows)); print("cols", cols[:20], "... n", len(cols))
    y, x = bad[0]; print("first", y, x, "got", got[y, x], "want", want[y, x])
