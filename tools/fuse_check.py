"""Quick K4 (fused single-pass) check on a GPU box: bit-exact parity against the oracle on random
shapes / windows / borders / bands / batches, then timings at 4096^2 with K4 on and off.
python tools/fuse_check.py [--quick] [--time-only]"""
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
    rng = np.random.default_rng(5)
    bad = 0
    kinds = {}
    for c in range(n):
        dtype = np.uint8 if c % 3 else np.uint16
        es = np.dtype(dtype).itemsize
        w, h = int(rng.integers(1, 1500)), int(rng.integers(1, 700))
        gx, gy = int(rng.integers(4, 60)), int(rng.integers(4, 60))
        wx, wy = 2 * gx + 1, 2 * gy + 1
        op = int(rng.integers(0, 2))
        border = int(rng.integers(0, 2))
        bval = int(rng.integers(0, int(np.iinfo(dtype).max) + 1))
        pad = (-w) % (16 // es) + (16 // es) * int(rng.integers(0, 2))
        img = R.generate(w, h, 100 + c, dtype=dtype)
        want = R.morph(img, wx, wy, op, border, bval)
        name = pkg.plan_name(es, w, h, wx, wy, op)
        kinds[name.split("_")[0]] = kinds.get(name.split("_")[0], 0) + 1
        if c % 4 == 3 and h > 8:  # row band with halos
            r0, r1 = h // 3, max(h // 3 + 1, 2 * h // 3)
            a, z = max(0, r0 - gy), min(h, r1 + gy)
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
            got = to_host(dst)
            ok = np.array_equal(got, want)
            if not ok:
                d = np.argwhere(got != want)
                print("  first diffs", d[:5].tolist(), "n", len(d))
        if not ok:
            bad += 1
            print("MISMATCH", c, dtype.__name__, w, h, wx, wy, op, border, bval, pad, name)
    print(f"parity: {n - bad}/{n} ok; planners {kinds}")
    return bad


def timing():
    for (wx, wy) in [(15, 15), (31, 31), (63, 63), (101, 101), (9, 9)]:
        for fuse in (1, 0):
            env = dict(os.environ, RMGPU_FUSE=str(fuse))
            out = subprocess.run([sys.executable, "tools/time_morph.py", "4096", "4096", str(wx), str(wy), "0", "1"],
                                 capture_output=True, text=True, env=env)
            print(("fuse " if fuse else "K3   ") + (out.stdout.strip() or out.stderr[-400:]))


if __name__ == "__main__":
    torch.cuda.set_device(0)
    bad = 0
    if "--time-only" not in sys.argv:
        bad = parity(40 if "--quick" in sys.argv else 200)
    timing()
    sys.exit(1 if bad else 0)
