"""Generates the committed golden fixtures in tests/golden/ (run in the build container, where
/root/reference is mounted and oracle/_ref/librmref.so -- the reference's own code -- is built).

  ref_u8.npz   outputs of the UNMODIFIED reference (rectmorph::erode/dilate/opening/closing/
               gradient, transpose_image, transpose_tile, linear_window_1d, van_herk_1d) on
               seeded inputs from the shared counter-based generator.
  u16.npz      16-bit cases: the reference has no u16 code, so these are the restatement's
               outputs, each asserted equal to OpenCV 4.13 (cv2.erode/dilate/morphologyEx on
               uint16 with the matching border) at generation time -- an independent pin.

Usage: python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402

OPS = {0: "erode", 1: "dilate", 2: "opening", 3: "closing", 4: "gradient"}


def u8_cases(R, F):
    rng = np.random.default_rng(20261020)
    arrays, meta = {}, []
    shapes = [(1, 1), (1, 9), (9, 1), (3, 3), (16, 16), (17, 5), (5, 33), (64, 48), (70, 70), (31, 97), (128, 3)]
    k = 0
    for (h, w) in shapes:
        for rep in range(6):
            wx = int(2 * rng.integers(0, 16) + 1)
            wy = int(2 * rng.integers(0, 16) + 1)
            op = int(rng.integers(0, 5))
            border = int(rng.integers(0, 2))
            bval = int(rng.integers(0, 256)) if border else 0
            seed = 1000 + k
            img = R.generate(w, h, seed, stream=0)
            out = F.morph(img, wx, wy, op, border, bval)
            arrays[f"in{k}"] = img
            arrays[f"out{k}"] = out
            meta.append(dict(case=k, w=w, h=h, wx=wx, wy=wy, op=op, border=border, bval=bval, seed=seed))
            k += 1
    # transposes via the reference
    for j, (h, w) in enumerate([(2, 3), (16, 16), (17, 33), (40, 7)]):
        img = R.generate(w, h, 5000 + j)
        arrays[f"tin{j}"] = img
        arrays[f"tout{j}"] = F.transpose_image(img)
    for n in (4, 8, 16):
        for dt in (np.uint8, np.uint16, np.uint32):
            t = (np.arange(n * n * 3, dtype=np.uint64) * 2654435761 % (1 << 32)).astype(dt)
            ref = t.copy()
            for i in range(3):
                view = ref[i * n * n:(i + 1) * n * n]
                F.transpose_tile(view, n, n)
            arrays[f"tile_in_{n}_{np.dtype(dt).name}"] = t
            arrays[f"tile_out_{n}_{np.dtype(dt).name}"] = ref
    # 1-D kernels with comparison counts
    one_d = []
    for j, (n, w) in enumerate([(8, 3), (50, 7), (64, 129), (10000, 31), (10000, 301)]):
        sig = R.generate(n, 1, 7000 + j)[0]
        for algo in (1, 2):
            for op in (0, 1):
                out, cnt = F.window_1d(sig, w, op, 0, 0, algo)
                arrays[f"d1_{j}_{algo}_{op}"] = out
                one_d.append(dict(j=j, n=n, w=w, algo=algo, op=op, comparisons=int(cnt), seed=7000 + j))
        arrays[f"d1in_{j}"] = sig
    return arrays, dict(morph=meta, one_d=one_d)


def u16_cases(R):
    import cv2
    rng = np.random.default_rng(4)
    arrays, meta = {}, []
    bt = {0: cv2.BORDER_REPLICATE, 1: cv2.BORDER_CONSTANT}
    for k in range(24):
        h, w = int(rng.integers(1, 60)), int(rng.integers(1, 60))
        wx, wy = int(2 * rng.integers(0, 12) + 1), int(2 * rng.integers(0, 12) + 1)
        op = int(rng.integers(0, 5))
        border = int(rng.integers(0, 2))
        bval = int(rng.integers(0, 65536)) if border else 0
        img = R.generate(w, h, 400 + k, stream=k, dtype=np.uint16)
        out = R.morph(img, wx, wy, op, border, bval)
        kern = np.ones((wy, wx), np.uint8)
        kw = dict(borderType=bt[border], borderValue=bval)
        er = lambda a: cv2.erode(a, kern, **kw)  # noqa: E731
        di = lambda a: cv2.dilate(a, kern, **kw)  # noqa: E731
        cv = {0: lambda a: er(a), 1: lambda a: di(a), 2: lambda a: di(er(a)), 3: lambda a: er(di(a)),
              4: lambda a: (di(a).astype(np.int64) - er(a)).astype(np.uint16)}[op](img)
        assert np.array_equal(cv, out), f"u16 restatement disagrees with OpenCV on case {k}"
        arrays[f"in{k}"] = img
        arrays[f"out{k}"] = out
        meta.append(dict(case=k, w=w, h=h, wx=wx, wy=wy, op=op, border=border, bval=bval, seed=400 + k,
                         stream=k))
    return arrays, dict(morph=meta)


def main():
    oracle.build()
    R, F = oracle.restatement(), oracle.reference()
    a8, m8 = u8_cases(R, F)
    np.savez_compressed(os.path.join(HERE, "ref_u8.npz"), **a8)
    a16, m16 = u16_cases(R)
    np.savez_compressed(os.path.join(HERE, "u16.npz"), **a16)
    gen = {"u8_seed7_64": R.generate(64, 1, 7)[0].tolist(),
           "u16_seed9_stream3_16": R.generate(16, 1, 9, stream=3, dtype=np.uint16)[0].tolist()}
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(dict(u8=m8, u16=m16, generator=gen,
                       note="ref_u8.npz from oracle/_ref (reference code); u16.npz from the restatement, "
                            "each case asserted equal to OpenCV 4.13 at generation time"), f, indent=1)
    print("wrote", sorted(os.listdir(HERE)))


if __name__ == "__main__":
    main()
