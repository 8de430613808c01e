"""K5 (chained passes in one persistent launch) check on a GPU box: bit-exact parity against the
oracle on random whole-image shapes / windows / borders / batches with the chain on, then timings
with the chain on and off.
python tools/chain_check.py [--quick] [--time-only] [--big]"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
import paper_2002_09474_b200 as pkg
from tests.gpu_util import empty_device, to_device, to_host

R = oracle.restatement()


def parity(n):
    rng = np.random.default_rng(9)
    bad = 0
    pkg.debug_set("chain", 1)
    for c in range(n):
        dtype = np.uint8 if c % 3 else np.uint16
        es = np.dtype(dtype).itemsize
        w, h = int(rng.integers(1, 2500)), int(rng.integers(64, 900))
        gx, gy = int(rng.integers(4, 60)), int(rng.integers(4, 60))
        wx, wy = 2 * gx + 1, 2 * gy + 1
        op = int(rng.integers(0, 4))  # erode, dilate, open, close
        border = int(rng.integers(0, 2))
        bval = int(rng.integers(0, int(np.iinfo(dtype).max) + 1))
        pad = (-w) % (16 // es) + (16 // es) * int(rng.integers(0, 2))
        batch = 1 if c % 5 else int(rng.integers(2, 5))
        imgs = [R.generate(w, h, 100 + c * 7 + b, dtype=dtype) for b in range(batch)]
        wants = [R.morph(im, wx, wy, op, border, bval) for im in imgs]
        before = pkg.launch_count()
        if batch == 1:
            src = to_device(imgs[0], pad)
            dst = empty_device(imgs[0].shape, dtype, pad)
            pkg.morph_device(src, dst, wx, wy, op, border, bval)
            torch.cuda.synchronize()
            gots = [to_host(dst)]
        else:
            src = torch.stack([to_device(im, 0) for im in imgs]) if w * es % 16 == 0 else None
            if src is None:
                continue
            dst = torch.empty_like(src)
            pkg.morph_batched_device(src, dst, wx, wy, op, border, bval)
            torch.cuda.synchronize()
            gots = [dst[b].cpu().numpy() for b in range(batch)]
        nl = pkg.launch_count() - before
        ok = all(np.array_equal(g, wnt) for g, wnt in zip(gots, wants))
        if not ok:
            bad += 1
            d = np.argwhere(gots[0] != wants[0])
            print("MISMATCH", c, dtype.__name__, w, h, wx, wy, op, border, bval, pad, batch, "launches", nl,
                  "first", d[:4].tolist(), "n", len(d))
    pkg.debug_set("chain", -1)
    print(f"parity: {n - bad}/{n} ok")
    return bad


def timing(big):
    cases = [(4096, 4096, w, w, 1, 1) for w in (15, 31, 63, 101)]
    cases += [(4096, 4096, 21, 21, 0, 2)]
    if big:
        cases += [(16384, 16384, 63, 63, 1, 1), (32768, 32768, 63, 63, 1, 1)]
    for (W, H, wx, wy, op, elem) in cases:
        for chain in (1, 0):
            env = dict(os.environ, RMGPU_CHAIN=str(chain))
            out = subprocess.run([sys.executable, "tools/time_morph.py", str(W), str(H), str(wx), str(wy), str(op), str(elem)],
                                 capture_output=True, text=True, env=env)
            print(("chain " if chain else "K3    ") + (out.stdout.strip() or out.stderr[-400:]), flush=True)


def cfg4(n_img=512):
    """cfg4: opening 21x21 of n_img 1024^2 u16 images, chain on / off (events, 5 reps, 2 rotating sets)."""
    srcs = [torch.empty((n_img, 1024, 1024), dtype=torch.uint16, device="cuda") for _ in range(2)]
    for k, s in enumerate(srcs):
        for b in range(0, n_img, 64):
            pkg.generate_device(s[b].view(1024, 1024), 3 + k, b)
        s[1:] = s[0].flip(0)[: n_img - 1] if False else s[1:]
    dsts = [torch.empty_like(s) for s in srcs]
    for chain in (1, 0, 1, 0):
        pkg.debug_set("chain", chain)
        for i in range(2):
            pkg.morph_batched_device(srcs[i], dsts[i], 21, 21, 2)
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        for r in range(6):
            pkg.morph_batched_device(srcs[r % 2], dsts[r % 2], 21, 21, 2)
        ev[1].record()
        torch.cuda.synchronize()
        us = ev[0].elapsed_time(ev[1]) / 6 * 1e3
        px = n_img * 1024 * 1024
        print(f"cfg4 chain={chain}: {us:.1f} us  {px / us / 1e3:.0f} Gpix/s  {4 * px / us / 1e3 / 6549.1 * 100:.1f}% of HBM", flush=True)
    pkg.debug_set("chain", -1)


if __name__ == "__main__":
    torch.cuda.set_device(0)
    bad = 0
    if "--time-only" not in sys.argv:
        bad = parity(30 if "--quick" in sys.argv else 150)
    timing("--big" in sys.argv)
    if "--cfg4" in sys.argv:
        cfg4()
    sys.exit(1 if bad else 0)
