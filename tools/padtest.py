import sys, os
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2002_09474_b200 as pkg
from tests.gpu_util import to_device, empty_device, to_host_full
import oracle
R = oracle.restatement()
for dtype in (np.uint8, np.uint16):
    img = R.generate(333, 97, 5, dtype=dtype)
    for pad in (3, 16, 61):
        src = to_device(img, pad, 0)
        dst = empty_device(img.shape, dtype, pad, 0xA5)
        pkg.morph_device(src, dst, 7, 5, 0)
        torch.cuda.synchronize()
        full = to_host_full(dst, 333 + pad)
        badc = np.where(np.any(full[:, 333:] != 0xA5, axis=0))[0]
        badr = np.where(np.any(full[:, 333:] != 0xA5, axis=1))[0]
        print(dtype.__name__, pad, "bad cols", badc[:10] + 333, "bad rows", badr[:10], len(badr), pkg.plan_name(img.itemsize, 333, 97, 7, 5, 0))
