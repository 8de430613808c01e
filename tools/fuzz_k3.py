"""Long randomized parity run of the separable K3 path against the C restatement (test-only oracle):
random shapes, windows, ops, borders, dtypes and planner knobs for a time budget.
python tools/fuzz_k3.py [seconds] [seed]"""
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
KNOBS = [{}, {"sep_vwarps": 8}, {"sep_hfirst": 0}, {"sep_strip": 0}, {"sep_vbulk": 1}, {"sep_notma": 0}, {"sep_hh": 2},
         {"sep_hh": 0}, {"sep_parts": 3}, {"sep_rb": 16}, {"sep_pdl": 1}, {"sep_c16_short": 0}]
t0, n, bad = time.time(), 0, 0
while time.time() - t0 < budget:
    knobs = KNOBS[int(rng.integers(0, len(KNOBS)))]
    for k, v in knobs.items():
        pkg.debug_set(k, v)
    dtype = np.uint8 if rng.random() < 0.7 else np.uint16
    es = np.dtype(dtype).itemsize
    w, h = int(rng.integers(1, 2500)), int(rng.integers(1, 900))
    gx = 0 if rng.random() < 0.15 else int(rng.integers(4, 70))
    gy = 0 if (gx and rng.random() < 0.15) else int(rng.integers(4, 70))
    op = int(rng.integers(0, 5))
    border = int(rng.integers(0, 2))
    bval = int(rng.integers(0, int(np.iinfo(dtype).max) + 1))
    img = R.generate(w, h, int(rng.integers(0, 1 << 30)), dtype=dtype)
    pad = (-w) % (16 // es) + (16 // es) * int(rng.integers(0, 2))
    src = to_device(img, pad)
    dst = empty_device(img.shape, dtype, pad)
    pkg.morph_device(src, dst, 2 * gx + 1, 2 * gy + 1, op, border, bval)
    torch.cuda.synchronize()
    want = R.morph(img, 2 * gx + 1, 2 * gy + 1, op, border, bval)
    if not np.array_equal(to_host(dst), want):
        bad += 1
        print("MISMATCH", knobs, dtype.__name__, w, h, 2 * gx + 1, 2 * gy + 1, op, border, bval, flush=True)
    for k in knobs:
        pkg.debug_set(k, -1)
    n += 1
print(f"fuzz_k3: {n} cases, {bad} mismatches in {time.time() - t0:.0f} s")
sys.exit(1 if bad else 0)
