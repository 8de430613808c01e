"""Randomized parity run of the small-window kernel K1 (windows <= 7 per axis) against the C
restatement (test-only oracle): random shapes, windows, ops (incl. gradient), borders, dtypes,
pitches, batches and row bands for a time budget. python tools/fuzz_k1.py [seconds] [seed]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2002_09474_b200 as pkg  # noqa: E402
from tests.gpu_util import empty_device, to_device, to_host  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
R = oracle.restatement()
t0, n, bad, used = time.time(), 0, 0, {}
while time.time() - t0 < budget:
    dtype = np.uint8 if rng.integers(0, 3) else np.uint16
    es = np.dtype(dtype).itemsize
    big = rng.integers(0, 8) == 0
    w = int(rng.integers(1, 5000 if big else 1400))
    h = int(rng.integers(1, 1200 if big else 300))
    wx, wy = 2 * int(rng.integers(0, 4)) + 1, 2 * int(rng.integers(0, 4)) + 1
    op = int(rng.integers(0, 5))
    border = int(rng.integers(0, 2))
    bval = int(rng.integers(0, int(np.iinfo(dtype).max) + 1))
    pad = (-w) % (16 // es) + (16 // es) * int(rng.integers(0, 3))
    img = R.generate(w, h, 1000 + n, dtype=dtype)
    want = R.morph(img, wx, wy, op, border, bval)
    kind = int(rng.integers(0, 3))
    halo = (wy // 2) * (2 if op in (2, 3) else 1)
    if kind == 1 and h > 8:
        r0, r1 = h // 3, max(h // 3 + 1, 2 * h // 3)
        a, z = max(0, r0 - halo), min(h, r1 + halo)
        src = to_device(img[a:z], pad)
        dst = empty_device((r1 - r0, w), dtype, pad)
        pkg.morph_band_device(src, r0 - a, z - r1, dst, wx, wy, op, border, bval)
        torch.cuda.synchronize()
        ok = np.array_equal(to_host(dst), want[r0:r1])
    else:
        src = to_device(img, pad)
        dst = empty_device(img.shape, dtype, pad)
        pkg.morph_device(src, dst, wx, wy, op, border, bval)
        torch.cuda.synchronize()
        ok = np.array_equal(to_host(dst), want)
    name = (pkg.plan_name(es, w, h, wx, wy, op) or "?").split("_")[0]
    used[name] = used.get(name, 0) + 1
    n += 1
    if not ok:
        bad += 1
        print("MISMATCH", dtype.__name__, w, h, wx, wy, op, border, bval, pad, kind, flush=True)
print(f"fuzz_k1: {n} cases, {bad} mismatches in {time.time() - t0:.0f} s; planners {used}")
sys.exit(1 if bad else 0)
