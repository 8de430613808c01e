"""GPU parity suite (-m gpu): the CUDA path through the C-ABI against the pinned oracle.

Bar: bit-exact (integer min/max and byte moves). Cases mirror the reference's acceptance
criteria 1, 2, 3, 5, 6 (proj/tests/acceptance.cpp:49-325) with the GPU entry points substituted,
plus GPU-specific layers: poisoned pitch padding, degenerate shapes, windows larger than the
image, batches, row bands with halos, and the BASELINE configs at full size.
"""
import json
import os
import subprocess

import numpy as np
import pytest

import oracle
from oracle import CLOSE, CONSTANT, DILATE, ERODE, GRADIENT, OPEN, REPLICATE
from tests.gpu_util import empty_device, to_device, to_host, to_host_full

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def gpu_morph(pkg, img, wx, wy, op, border=REPLICATE, bval=0, pad=0, poison=None):
    src = to_device(img, pad, poison)
    dst = empty_device(img.shape, img.dtype, pad, 0xA5 if poison is not None else 0)
    pkg.morph_device(src, dst, wx, wy, op, border, bval)
    return to_host(dst), dst


def test_golden_u8_reference_outputs(gpu):
    meta = json.load(open(os.path.join(GOLDEN, "golden.json")))["u8"]
    z = np.load(os.path.join(GOLDEN, "ref_u8.npz"))
    for c in meta["morph"]:
        img = z[f"in{c['case']}"]
        got, _ = gpu_morph(gpu, img, c["wx"], c["wy"], c["op"], c["border"], c["bval"])
        assert np.array_equal(got, z[f"out{c['case']}"]), c
        # the host-buffer (drop-in) entry point must agree too
        host = {0: gpu.erode, 1: gpu.dilate, 2: gpu.opening, 3: gpu.closing, 4: gpu.gradient}[c["op"]](
            img, gpu.StructuringElement(c["wx"], c["wy"]), gpu.BorderPolicy(c["border"], c["bval"]))
        assert np.array_equal(host, z[f"out{c['case']}"]), c
    for j in range(4):
        assert np.array_equal(gpu.transpose_image(z[f"tin{j}"]), z[f"tout{j}"])
    for n in (4, 8, 16):
        for dt in ("uint8", "uint16", "uint32"):
            t = z[f"tile_in_{n}_{dt}"].copy()
            for i in range(3):
                gpu.transpose_tile(t, n, n, offset=i * n * n)
            assert np.array_equal(t, z[f"tile_out_{n}_{dt}"]), (n, dt)
    for d in meta["one_d"]:
        f = gpu.van_herk_1d if d["algo"] == 2 else gpu.linear_window_1d
        cnt = gpu.api.OpCounter()
        out = f(z[f"d1in_{d['j']}"], d["w"], gpu.OpKind(d["op"]), counter=cnt)
        assert np.array_equal(out, z[f"d1_{d['j']}_{d['algo']}_{d['op']}"])
        assert cnt.comparisons == d["comparisons"]


def test_golden_u16(gpu):
    meta = json.load(open(os.path.join(GOLDEN, "golden.json")))["u16"]
    z = np.load(os.path.join(GOLDEN, "u16.npz"))
    for c in meta["morph"]:
        img = z[f"in{c['case']}"]
        got, _ = gpu_morph(gpu, img, c["wx"], c["wy"], c["op"], c["border"], c["bval"])
        assert np.array_equal(got, z[f"out{c['case']}"]), c


def test_known_answers(gpu):
    img = np.array([[9, 8, 7], [6, 5, 4], [3, 2, 1]], np.uint8)
    assert gpu.erode(img, gpu.make_se(3, 3)).tolist() == [[5, 4, 4], [2, 1, 1], [2, 1, 1]]
    sig = np.array([4, 2, 6, 1, 3, 5, 0, 7], np.uint8)
    assert gpu.linear_window_1d(sig, 3, gpu.OpKind.Erode).tolist() == [2, 2, 1, 1, 1, 0, 0, 0]
    assert gpu.van_herk_1d(sig, 3, gpu.OpKind.Dilate).tolist() == [4, 6, 6, 6, 5, 5, 7, 7]
    sq = np.full((2, 2), 128, np.uint8)
    assert np.all(gpu.erode(sq, gpu.make_se(3, 3), gpu.BorderPolicy.constant(5)) == 5)
    assert np.all(gpu.dilate(sq, gpu.make_se(3, 3), gpu.BorderPolicy.constant(200)) == 200)
    assert gpu.transpose_image(np.array([[1, 2, 3], [4, 5, 6]], np.uint8)).ravel().tolist() == [1, 4, 2, 5, 3, 6]


@pytest.mark.parametrize("dtype", [np.uint8, np.uint16])
def test_exhaustive_small(gpu, restatement, dtype):
    # acceptance criterion 1 (acceptance.cpp:49-93): sizes 1..16 x SE up to 9x9 x ops x borders
    mx = np.iinfo(dtype).max
    for w in range(1, 17):
        for h in range(1, 17, 2):
            img = restatement.generate(w, h, w * 64 + h, dtype=dtype)
            for sw in (1, 3, 5, 7, 9):
                for sh in (1, 3, 9):
                    for op in (ERODE, DILATE):
                        for border, bval in ((REPLICATE, 0), (CONSTANT, mx if op == ERODE else 0), (CONSTANT, 77)):
                            want = restatement.morph(img, sw, sh, op, border, bval)
                            got, _ = gpu_morph(gpu, img, sw, sh, op, border, bval)
                            assert np.array_equal(got, want), (w, h, sw, sh, op, border, bval)


@pytest.mark.parametrize("dtype", [np.uint8, np.uint16])
def test_random_medium_all_ops(gpu, restatement, dtype):
    # acceptance criterion 2 (acceptance.cpp:97-132) widened to every op and border
    rng = np.random.default_rng(20260815)
    mx = int(np.iinfo(dtype).max)
    for c in range(150):
        w, h = (int(v) for v in rng.integers(1, 200, 2))
        wx, wy = (int(2 * v + 1) for v in rng.integers(0, 40, 2))
        op = int(rng.integers(0, 5))
        border = int(rng.integers(0, 2))
        bval = int(rng.integers(0, mx + 1))
        pad = int(rng.integers(0, 3)) * 16 // np.dtype(dtype).itemsize + int(rng.integers(0, 5))
        img = restatement.generate(w, h, 7000 + c, dtype=dtype)
        want = restatement.morph(img, wx, wy, op, border, bval)
        got, _ = gpu_morph(gpu, img, wx, wy, op, border, bval, pad=pad)
        assert np.array_equal(got, want), (c, w, h, wx, wy, op, border, bval)


@pytest.mark.parametrize("dtype", [np.uint8, np.uint16])
def test_small_window_fuzz_aligned(gpu, restatement, dtype):
    # windows <= 7 on 16-byte aligned pitches: the register-streaming kernel (col_*) -- strip
    # edges, image edges, widths around the 512-byte strip, short / tall images, both borders
    rng = np.random.default_rng(4242 + np.dtype(dtype).itemsize)
    mx = int(np.iinfo(dtype).max)
    es = np.dtype(dtype).itemsize
    widths = [1, 3, 4, 15, 16, 17, 255, 256, 257, 300, 508, 511, 512, 513, 516, 517, 1023, 1024, 1030, 1500]
    seen = set()
    for c in range(120):
        w = int(widths[c % len(widths)]) if c < 60 else int(rng.integers(1, 1600))
        h = int(rng.integers(1, 90))
        wx, wy = (int(2 * v + 1) for v in rng.integers(0, 4, 2))
        op = int(rng.integers(0, 2))
        border = int(rng.integers(0, 2))
        bval = int(rng.integers(0, mx + 1))
        pad = (-w) % (16 // es) + int(rng.integers(0, 3)) * (16 // es)
        img = restatement.generate(w, h, 9100 + c, dtype=dtype)
        want = restatement.morph(img, wx, wy, op, border, bval)
        got, dst = gpu_morph(gpu, img, wx, wy, op, border, bval, pad=pad, poison=0x5A)
        assert np.array_equal(got, want), (c, w, h, wx, wy, op, border, bval, pad)
        full = to_host_full(dst, w + pad)
        assert np.all(full[:, w:] == 0xA5), ("padding written", c, w, h, wx, wy)
        seen.add(gpu.plan_name(es, w, h, wx, wy, op).split("_")[0])
    assert "col" in seen, seen


@pytest.mark.parametrize("win", [(3, 3), (7, 7), (15, 15), (21, 21), (31, 31), (63, 63), (101, 101), (31, 1),
                                 (1, 31), (151, 5), (5, 151), (301, 301), (1001, 3)])
def test_window_sweep(gpu, restatement, win):
    wx, wy = win
    for dtype in (np.uint8, np.uint16):
        img = restatement.generate(517, 389, wx * 1000 + wy, dtype=dtype)
        for op in (ERODE, DILATE):
            want = restatement.morph(img, wx, wy, op, REPLICATE, 0)
            got, _ = gpu_morph(gpu, img, wx, wy, op)
            assert np.array_equal(got, want), (win, dtype, op)
        want = restatement.morph(img, wx, wy, DILATE, CONSTANT, 3)
        got, _ = gpu_morph(gpu, img, wx, wy, DILATE, CONSTANT, 3)
        assert np.array_equal(got, want)


def test_degenerate_shapes(gpu, restatement):
    for (h, w) in [(1, 1), (1, 2), (2, 1), (1, 4097), (4097, 1), (3, 1000), (1000, 3), (17, 15)]:
        for dtype in (np.uint8, np.uint16):
            img = restatement.generate(w, h, h * 7 + w, dtype=dtype)
            for wx, wy in [(3, 3), (9, 1), (1, 9), (2 * w + 5, 2 * h + 3), (101, 101)]:
                for op in (ERODE, DILATE, OPEN, CLOSE, GRADIENT):
                    for border, bval in ((REPLICATE, 0), (CONSTANT, 9)):
                        want = restatement.morph(img, wx, wy, op, border, bval)
                        got, _ = gpu_morph(gpu, img, wx, wy, op, border, bval)
                        assert np.array_equal(got, want), (h, w, wx, wy, op, border)


def test_padding_never_leaks_or_is_written(gpu, restatement):
    # test_separable.cpp:214-229 / test_transpose.cpp:145-157 on device: poisoned pitch padding
    for dtype in (np.uint8, np.uint16):
        img = restatement.generate(333, 97, 5, dtype=dtype)
        want = restatement.morph(img, 7, 5, ERODE)
        for pad in (3, 16, 61):
            got, dst = gpu_morph(gpu, img, 7, 5, ERODE, pad=pad, poison=0)
            assert np.array_equal(got, want)
            full = to_host_full(dst, 333 + pad)
            assert np.all(full[:, 333:] == (0xA5 if dtype == np.uint8 else 0xA5)), "padding written"


def test_algebraic_properties(gpu, restatement):
    # acceptance criterion 6 (acceptance.cpp:275-325) on the GPU results
    se = gpu.make_se(5, 5)
    for seed in range(20):
        a = restatement.generate(32, 32, 11000 + seed)
        e, d = gpu.erode(a, se), gpu.dilate(a, se)
        assert np.array_equal(d, 255 - gpu.erode(255 - a, se))
        assert np.all(e <= a) and np.all(a <= d)
        o, c = gpu.opening(a, se), gpu.closing(a, se)
        assert np.array_equal(gpu.opening(o, se), o)
        assert np.array_equal(gpu.closing(c, se), c)
        assert np.array_equal(gpu.gradient(a, se), d - e)
        b = np.maximum(a, restatement.generate(32, 32, 12000 + seed))
        assert np.all(e <= gpu.erode(b, se)) and np.all(d <= gpu.dilate(b, se))


@pytest.mark.parametrize("op", [ERODE, DILATE, OPEN, CLOSE, GRADIENT])
def test_batched(gpu, restatement, op):
    import torch
    for dtype in (np.uint8, np.uint16):
        imgs = np.stack([restatement.generate(129, 67, 40 + b, stream=b, dtype=dtype) for b in range(5)])
        src = to_device(imgs, 8)
        dst = empty_device(imgs.shape, dtype, 8)
        gpu.morph_batched_device(src, dst, 21, 9, op)
        torch.cuda.synchronize()
        got = to_host(dst)
        for b in range(5):
            assert np.array_equal(got[b], restatement.morph(imgs[b], 21, 9, op)), (b, dtype)


@pytest.mark.parametrize("op", [ERODE, DILATE, OPEN, CLOSE, GRADIENT])
def test_row_bands_with_halo(gpu, restatement, op):
    # the multi-GPU row decomposition on one device: each band + its halo rows -> exact rows
    for dtype in (np.uint8, np.uint16):
        H, W, wx, wy = 203, 150, 7, 15
        img = restatement.generate(W, H, 77, dtype=dtype)
        for border, bval in ((REPLICATE, 0), (CONSTANT, 200)):
            want = restatement.morph(img, wx, wy, op, border, bval)
            halo = (wy // 2) * (2 if op in (OPEN, CLOSE) else 1)
            for nb in (1, 2, 3, 7):
                out = np.zeros_like(img)
                for k in range(nb):
                    r0, r1 = H * k // nb, H * (k + 1) // nb
                    a, z = max(0, r0 - halo), min(H, r1 + halo)
                    src = to_device(img[a:z], 5)
                    dst = empty_device((r1 - r0, W), dtype, 3)
                    gpu.morph_band_device(src, r0 - a, z - r1, dst, wx, wy, op, border, bval)
                    out[r0:r1] = to_host(dst)
                assert np.array_equal(out, want), (op, dtype, border, nb)


@pytest.mark.parametrize("dtype", [np.uint8, np.uint16])
def test_aligned_batches_and_bands_fuzz(gpu, restatement, dtype):
    # 16-byte aligned pitches and image strides, so batches and row bands (explicit halo rows)
    # go through the TMA kernels (K1 for w <= 7, K2 otherwise): every op, both borders
    import torch
    rng = np.random.default_rng(99 + np.dtype(dtype).itemsize)
    mx = int(np.iinfo(dtype).max)
    es = np.dtype(dtype).itemsize
    kinds = set()
    for c in range(120):
        w = int(rng.integers(1, 700))
        h = int(rng.integers(1, 300))
        small = c % 2 == 0
        wx = int(2 * rng.integers(0, 4 if small else 40) + 1)
        wy = int(2 * rng.integers(0, 4 if small else 40) + 1)
        op = int(rng.integers(0, 5))
        border = int(rng.integers(0, 2))
        bval = int(rng.integers(0, mx + 1))
        pad = (-w) % (16 // es)
        if c % 4 < 2:  # batch of independent images
            nb = int(rng.integers(2, 5))
            imgs = np.stack([restatement.generate(w, h, 500 + 10 * c + b, stream=b, dtype=dtype) for b in range(nb)])
            src = to_device(imgs, pad)
            dst = empty_device(imgs.shape, dtype, pad)
            gpu.morph_batched_device(src, dst, wx, wy, op, border, bval)
            torch.cuda.synchronize()
            got = to_host(dst)
            for b in range(nb):
                want = restatement.morph(imgs[b], wx, wy, op, border, bval)
                assert np.array_equal(got[b], want), ("batch", c, b, w, h, wx, wy, op, border)
        else:  # row bands with real halo rows, as the multi-GPU split uses them
            img = restatement.generate(w, h, 900 + c, dtype=dtype)
            want = restatement.morph(img, wx, wy, op, border, bval)
            halo = (wy // 2) * (2 if op in (OPEN, CLOSE) else 1)
            nbands = int(rng.integers(1, 5))
            out = np.zeros_like(img)
            for k in range(nbands):
                r0, r1 = h * k // nbands, h * (k + 1) // nbands
                if r1 == r0:
                    continue
                a, z = max(0, r0 - halo), min(h, r1 + halo)
                src = to_device(img[a:z], pad)
                dst = empty_device((r1 - r0, w), dtype, pad)
                gpu.morph_band_device(src, r0 - a, z - r1, dst, wx, wy, op, border, bval)
                out[r0:r1] = to_host(dst)
            assert np.array_equal(out, want), ("bands", c, w, h, wx, wy, op, border, nbands)
        kinds.add(gpu.plan_name(es, w, h, wx, wy, op).split("_")[0])
    assert {"col", "sep"} <= kinds, kinds


SEP_KNOBS = [
    {},                                   # planner defaults
    {"sep_notma": 0, "sep_pf": 1},        # TMA-fed vertical pass on small images (one slot ahead)
    {"sep_notma": 0, "sep_pf": 3, "sep_rb": 24},  # deeper TMA prefetch, short bands (more edge bands)
    {"sep_notma": 1, "sep_rb": 8},        # plain-load vertical pass, one block per band
    {"sep_l2mb": 0, "sep_parts": 3, "sep_hfirst": 0},  # vertical pass first, 64-row L2 bands, 3 parts
    {"sep_parts": 1, "sep_pdl": 1, "sep_hfirst": 0},  # one warp per row group, PDL between passes, V first
    {"sep_pdl": 1},                       # PDL between the passes, H first
    {"sep_hh": 0},                        # opening / closing as four passes
    {"sep_hh": 2},                        # opening / closing always in three (also 16-column chunks)
    {"sep_c16_short": 0},                 # u8 wings 4..7 in 8-column chunks (else half-chunk scans)
    {"sep_strip": 0},                     # H first into a row-major intermediate (not strip-major)
    {"sep_vbulk": 1, "sep_pf": 2},        # strip-major intermediate read by 1-D bulk copies (TMA pipeline)
]


@pytest.mark.parametrize("knobs", [{}, {"sep_notma": 0}, {"sep_hfirst": 0, "sep_notma": 0}, {"sep_vbulk": 1}])
def test_sep_large_shapes(gpu, restatement, knobs):
    # K3 on images wide and tall enough for many strips, column parts and row bands (both pass
    # orders; the TMA vertical pass forced on), ragged widths, every op, both borders
    rng = np.random.default_rng(4242 + len(knobs))
    for k, v in knobs.items():
        gpu.debug_set(k, v)
    try:
        for c in range(6):
            dtype = np.uint8 if c % 3 else np.uint16
            es = np.dtype(dtype).itemsize
            w, h = int(rng.integers(1500, 4200)), int(rng.integers(300, 1300))
            g = int(rng.integers(4, 60))
            wx, wy = 2 * g + 1, 2 * int(rng.integers(4, 60)) + 1
            op, border = c % 5, int(rng.integers(0, 2))
            bval = int(rng.integers(0, int(np.iinfo(dtype).max) + 1))
            img = restatement.generate(w, h, 7000 + c, dtype=dtype)
            got, _ = gpu_morph(gpu, img, wx, wy, op, border, bval, (-w) % (16 // es))
            assert np.array_equal(got, restatement.morph(img, wx, wy, op, border, bval)), (knobs, c, w, h, wx, wy, op)
    finally:
        for k in knobs:
            gpu.debug_set(k, -1)


@pytest.mark.parametrize("dtype", [np.uint8, np.uint16])
def test_phase_kernel_fuzz(gpu, restatement, dtype):
    # K2 (persistent phase kernel) with K3 switched off: it stays the path for windows K3 declines
    # (one wing in 1..3 with the other large, wings past K3's register budget) and must stay exact
    rng = np.random.default_rng(77 + np.dtype(dtype).itemsize)
    mx = int(np.iinfo(dtype).max)
    es = np.dtype(dtype).itemsize
    gpu.debug_set("sep", 0)
    try:
        seen = set()
        for c in range(40):
            w, h = int(rng.integers(1, 700)), int(rng.integers(1, 300))
            wx = 2 * int(rng.integers(0, 50)) + 1
            wy = 2 * int(rng.integers(4, 50)) + 1 if c % 2 else 2 * int(rng.integers(0, 4)) + 1
            op, border, bval = int(rng.integers(0, 2)), int(rng.integers(0, 2)), int(rng.integers(0, mx + 1))
            pad = (-w) % (16 // es)
            img = restatement.generate(w, h, 40 + c, dtype=dtype)
            got, _ = gpu_morph(gpu, img, wx, wy, op, border, bval, pad)
            assert np.array_equal(got, restatement.morph(img, wx, wy, op, border, bval)), (c, w, h, wx, wy, op, border)
            seen.add(gpu.plan_name(es, w, h, wx, wy, op).split("_")[0])
        assert "phase" in seen, seen
    finally:
        gpu.debug_set("sep", -1)


@pytest.mark.parametrize("knobs", range(len(SEP_KNOBS)))
@pytest.mark.parametrize("dtype", [np.uint8, np.uint16])
def test_sep_passes_fuzz(gpu, restatement, dtype, knobs):
    # K3 (separable streaming passes through L2) under every planner knob that changes its launch
    # geometry: every chunk class g mod C, block size / tail r, edge bands, ragged words, batches
    # and row bands, both borders
    _planner_fuzz(gpu, restatement, dtype, knobs, dict(SEP_KNOBS[knobs]), "sep")


FUSE_KNOBS = [
    {"fuse": 1},                                  # K4 (single-pass fused kernel) with its defaults
    {"fuse": 1, "fuse_pf": 1, "fuse_nt": 2},      # one block of TMA prefetch, two tile slots
    {"fuse": 1, "fuse_pair": 1, "fuse_b": 12},    # one block per TMA box, 12-row blocks only
]


@pytest.mark.parametrize("knobs", range(len(FUSE_KNOBS)))
@pytest.mark.parametrize("dtype", [np.uint8, np.uint16])
def test_fused_kernel_fuzz(gpu, restatement, dtype, knobs):
    # K4 (vertical and horizontal pass in one kernel, intermediate in shared memory; off by default)
    # on the same random images, batches and row bands; windows it declines stay on K3
    _planner_fuzz(gpu, restatement, dtype, 100 + knobs, dict(FUSE_KNOBS[knobs]), "fuse")


def _planner_fuzz(gpu, restatement, dtype, knobs, knob_set, expect):
    import torch
    rng = np.random.default_rng(1234 + 7 * knobs + np.dtype(dtype).itemsize)
    mx = int(np.iinfo(dtype).max)
    es = np.dtype(dtype).itemsize
    for k, v in knob_set.items():
        gpu.debug_set(k, v)
    try:
        seen = set()
        for c in range(48):
            w = int(rng.integers(1, 900))
            h = int(rng.integers(1, 400))
            g = [0, int(rng.integers(4, 70)), int(rng.integers(4, 20))]
            wx = 2 * g[int(rng.integers(0, 3))] + 1 if c % 6 else 2 * int(rng.integers(4, 16)) + 1
            wy = 2 * g[int(rng.integers(0, 3))] + 1 if c % 5 else 1
            if wx == 1 and wy == 1:
                wx = 2 * int(rng.integers(4, 40)) + 1
            op = int(rng.integers(0, 5))  # erode, dilate, opening, closing, gradient
            border = int(rng.integers(0, 2))
            bval = int(rng.integers(0, mx + 1))
            pad = (-w) % (16 // es) + 16 // es * int(rng.integers(0, 3))
            if c % 3 == 0:
                nb = int(rng.integers(2, 4))
                imgs = np.stack([restatement.generate(w, h, 70 + 10 * c + b, stream=b, dtype=dtype) for b in range(nb)])
                src = to_device(imgs, pad)
                dst = empty_device(imgs.shape, dtype, pad)
                gpu.morph_batched_device(src, dst, wx, wy, op, border, bval)
                torch.cuda.synchronize()
                got = to_host(dst)
                for b in range(nb):
                    want = restatement.morph(imgs[b], wx, wy, op, border, bval)
                    assert np.array_equal(got[b], want), ("batch", knobs, c, b, w, h, wx, wy, op, border)
            elif c % 3 == 1:
                img = restatement.generate(w, h, 300 + c, dtype=dtype)
                want = restatement.morph(img, wx, wy, op, border, bval)
                halo = (wy // 2) * (2 if op in (OPEN, CLOSE) else 1)
                r0, r1 = h // 3, max(h // 3 + 1, 2 * h // 3)
                a, z = max(0, r0 - halo), min(h, r1 + halo)
                src = to_device(img[a:z], pad)
                dst = empty_device((r1 - r0, w), dtype, pad)
                gpu.morph_band_device(src, r0 - a, z - r1, dst, wx, wy, op, border, bval)
                assert np.array_equal(to_host(dst), want[r0:r1]), ("band", knobs, c, w, h, wx, wy, op, border)
            else:
                img = restatement.generate(w, h, 600 + c, dtype=dtype)
                got, _ = gpu_morph(gpu, img, wx, wy, op, border, bval, pad)
                want = restatement.morph(img, wx, wy, op, border, bval)
                assert np.array_equal(got, want), ("image", knobs, c, w, h, wx, wy, op, border)
            seen.add(gpu.plan_name(es, w, h, wx, wy, op).split("_")[0])
        assert expect in seen, seen
    finally:
        for k in knob_set:
            gpu.debug_set(k, -1)


def test_transpose_images(gpu, restatement):
    import torch
    for dtype in (np.uint8, np.uint16):
        for (h, w) in [(1, 1), (2, 3), (64, 64), (65, 63), (100, 333), (1024, 4096 + 7)]:
            img = restatement.generate(w, h, h + w, dtype=dtype)
            src = to_device(img, 3)
            dst = empty_device((w, h), dtype, 5)
            gpu.transpose_device(src, dst)
            torch.cuda.synchronize()
            assert np.array_equal(to_host(dst), img.T), (dtype, h, w)
            assert np.array_equal(gpu.transpose_image(img), img.T)


def test_transpose_images_aligned(gpu, restatement):
    # 16-byte aligned pitches: full 64x64 tiles through the register-butterfly kernel, ragged
    # right / bottom strips through the shared-memory kernel
    import torch
    for dtype in (np.uint8, np.uint16):
        es = np.dtype(dtype).itemsize
        for (h, w) in [(64, 64), (128, 192), (100, 333), (65, 1000), (1000, 65), (512, 2048), (777, 1500)]:
            img = restatement.generate(w, h, 3 * h + w, dtype=dtype)
            src = to_device(img, (-w) % (16 // es) + 16 // es)
            dst = empty_device((w, h), dtype, (-h) % (16 // es), 0x3C)
            gpu.transpose_device(src, dst)
            torch.cuda.synchronize()
            assert np.array_equal(to_host(dst), img.T), (dtype, h, w)
            full = to_host_full(dst, h + (-h) % (16 // es))
            assert np.all(full[:, h:] == 0x3C), ("padding written", dtype, h, w)


def test_host_entry_pipelined_bands(gpu, restatement):
    # host-buffer entry point on images large enough to be pipelined in row bands (H2D / kernel /
    # D2H overlapped): identical to the device-buffer call on the whole image
    import torch
    for dtype, (w, h) in ((np.uint8, (4096, 2048)), (np.uint16, (1500, 1999))):
        img = restatement.generate(w, h, 77, dtype=dtype)
        mx = int(np.iinfo(dtype).max)
        for (wx, wy, op, border, bval) in [(3, 3, ERODE, REPLICATE, 0), (63, 63, DILATE, REPLICATE, 0),
                                           (21, 21, OPEN, CONSTANT, mx // 3), (5, 31, CLOSE, REPLICATE, 0),
                                           (7, 7, GRADIENT, CONSTANT, 9), (1, 101, ERODE, CONSTANT, mx)]:
            fn = {ERODE: gpu.erode, DILATE: gpu.dilate, OPEN: gpu.opening, CLOSE: gpu.closing,
                  GRADIENT: gpu.gradient}[op]
            got = fn(img, gpu.StructuringElement(wx, wy), gpu.BorderPolicy(border, bval))
            want, _ = gpu_morph(gpu, img, wx, wy, op, border, bval)
            assert np.array_equal(got, want), (dtype, wx, wy, op, border)


def test_host_entry_concurrent_callers(gpu, restatement):
    # several threads inside the synchronous host entry at once (ctypes drops the GIL): every call has
    # its own streams and graph cache, the band count follows the number of calls in flight, and a
    # sweep of more windows than the old 8-entry graph cache held still replays cached graphs
    import concurrent.futures as cf
    img = restatement.generate(4096, 2304, 91, dtype=np.uint8)  # >= 8 MB: pipelined when alone
    windows = [(3, 3), (7, 7), (15, 15), (31, 31), (63, 63), (101, 101), (31, 1), (1, 31), (9, 21), (5, 5)]
    jobs = [(wx, wy, op) for (wx, wy) in windows for op in (ERODE, DILATE)]
    want = {j: restatement.morph(img, j[0], j[1], j[2], REPLICATE, 0) for j in jobs}

    def run(j):
        fn = gpu.erode if j[2] == ERODE else gpu.dilate
        return j, fn(img, gpu.StructuringElement(j[0], j[1]), gpu.BorderPolicy(REPLICATE, 0))

    for workers in (3, 1):
        with cf.ThreadPoolExecutor(workers) as ex:
            for rep in range(2):  # the second sweep replays the cached graphs
                for j, got in ex.map(run, jobs):
                    assert np.array_equal(got, want[j]), (workers, rep, j)


def test_transpose_tiles(gpu, restatement):
    import torch
    for dt in (np.uint8, np.uint16, np.uint32):
        for n in (4, 8, 16):
            t = (restatement.generate(n * n * 300, 1, n, dtype=np.uint16)[0].astype(np.uint64) * 40503).astype(dt)
            want = restatement.transpose_tiles(t, n) if dt != np.uint32 else \
                np.ascontiguousarray(t.reshape(-1, n, n).transpose(0, 2, 1)).ravel()
            dev = torch.from_numpy(t.view(np.uint8).copy()).cuda()
            dv = dev.view({1: torch.uint8, 2: torch.uint16, 4: torch.int32}[t.itemsize])
            gpu.transpose_tiles_device(dv, n)
            torch.cuda.synchronize()
            got = dev.cpu().numpy().view(dt)
            assert np.array_equal(got, want), (dt, n)
            # strided tiles inside a wider buffer leave the neighbours untouched
            buf = (np.arange(n * (n + 3) * 4) * 7 % 251).astype(dt)
            ref = buf.copy()
            for i in range(4):
                v = ref[i * n * (n + 3):(i + 1) * n * (n + 3)].reshape(n, n + 3)
                v[:, :n] = v[:, :n].T.copy()
            dev = torch.from_numpy(buf.view(np.uint8).copy()).cuda()
            gpu.transpose_tiles_device(dev.view({1: torch.uint8, 2: torch.uint16, 4: torch.int32}[buf.itemsize]),
                                       n, n_tiles=4, row_stride=n + 3, tile_step=n * (n + 3))
            torch.cuda.synchronize()
            assert np.array_equal(dev.cpu().numpy().view(dt), ref)


def test_one_d_api(gpu, restatement):
    for n in (1, 2, 7, 64, 1000):
        sig = restatement.generate(n, 1, n)[0]
        for w in (1, 3, 31, 129):
            for op in (0, 1):
                for border, bval in ((REPLICATE, 0), (CONSTANT, 17)):
                    want, _ = restatement.window_1d(sig, w, op, border, bval)
                    b = gpu.BorderPolicy(border, bval)
                    assert np.array_equal(gpu.linear_window_1d(sig, w, gpu.OpKind(op), b), want)
                    assert np.array_equal(gpu.van_herk_1d(sig, w, gpu.OpKind(op), b), want)


def test_pass_api(gpu, reference):
    img = np.random.default_rng(3).integers(0, 256, (77, 131), dtype=np.uint8)
    for w in (1, 3, 17, 63):
        for op in (0, 1):
            assert np.array_equal(gpu.horizontal_pass(img, gpu.OpKind(op), w), reference.pass_(0, img, w, op))
            assert np.array_equal(gpu.vertical_pass_direct(img, gpu.OpKind(op), w), reference.pass_(1, img, w, op))
            assert np.array_equal(gpu.vertical_pass_via_transpose(img, gpu.OpKind(op), w),
                                  reference.pass_(2, img, w, op, algo=2))


def test_cfg2_full_size_against_reference(gpu, restatement, reference):
    # BASELINE cfg2 at full size: 4096^2 u8, every window of the sweep, both ops, exact against the
    # reference's own code (multi-threaded row bands, themselves pinned by test_oracle).
    import bench
    img = bench.cfg2_image()
    for wx, wy in bench.CFG2_WINDOWS:
        for op in (ERODE, DILATE):
            want = reference.morph(img, wx, wy, op, nthreads=os.cpu_count() or 4)
            got, _ = gpu_morph(gpu, img, wx, wy, op)
            assert np.array_equal(got, want), (wx, wy, op)


def test_cfg1_full_size(gpu, reference, restatement):
    img = restatement.generate(1920, 1080, 1)
    for op in (ERODE, DILATE):
        got, _ = gpu_morph(gpu, img, 3, 3, op)
        assert np.array_equal(got, reference.morph(img, 3, 3, op))


def test_cfg3_transposes_full_size(gpu, restatement):
    # BASELINE cfg3 at full size: 8192^2 u8 and u16 images and all 2^24 8x8 / 16x16 u8 tiles,
    # every element compared with the closed form (x^T; per tile t[i][j] <- t[j][i],
    # transpose.hpp:19-30), the inputs pinned to the generator the restatement shares
    import torch
    for dtype, seed in ((np.uint8, 3), (np.uint16, 30)):
        src = torch.empty((8192, 8192), dtype=torch.uint8 if dtype == np.uint8 else torch.uint16, device="cuda")
        gpu.generate_device(src, seed)
        dst = torch.empty_like(src)
        gpu.transpose_device(src, dst)
        torch.cuda.synchronize()
        s8 = src.view(torch.uint8).view(8192, 8192, -1)  # compare as bytes (uint16 eq needs no arithmetic)
        assert torch.equal(dst.view(torch.uint8).view(8192, 8192, -1), s8.transpose(0, 1).contiguous()), dtype
        assert np.array_equal(to_host(src[:4]), restatement.generate(8192, 4, seed, dtype=dtype))
    for n, seed in ((8, 31), (16, 32)):
        t = torch.empty(((1 << 24) * n * n // 4096, 4096), dtype=torch.uint8, device="cuda")
        gpu.generate_device(t, seed)
        want = t.view(-1, n, n).transpose(1, 2).contiguous()
        assert np.array_equal(to_host(t[:2]), restatement.generate(4096, 2, seed))
        gpu.transpose_tiles_device(t, n)
        torch.cuda.synchronize()
        assert torch.equal(t.view(-1, n, n), want), n
        del t, want
        torch.cuda.empty_cache()


def test_cfg4_opening_u16_full_batch(gpu, restatement):
    # BASELINE cfg4 at full size: all 512 u16 1024^2 images (seed 4, stream = image index), one
    # batched opening 21x21, every image compared with the restatement (host threads in parallel;
    # van Herk in the restatement for speed -- its algorithms are pinned equal in test_oracle)
    import concurrent.futures as cf
    import torch
    from oracle import VANHERK
    B, N = 512, 1024
    imgs = torch.empty((B, N, N), dtype=torch.uint16, device="cuda")
    for b in range(B):
        gpu.generate_device(imgs[b], 4, stream_id=b)
    out = torch.empty_like(imgs)
    gpu.morph_batched_device(imgs, out, 21, 21, OPEN)
    torch.cuda.synchronize()
    host = to_host(out)
    assert host.shape == (B, N, N)

    def check(b):
        src = restatement.generate(N, N, 4, stream=b, dtype=np.uint16)
        return b, np.array_equal(host[b], restatement.morph(src, 21, 21, OPEN, h_algo=VANHERK, v_algo=VANHERK))

    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 8) as ex:
        bad = [b for b, ok in ex.map(check, range(B)) if not ok]
    assert not bad, bad


def test_cfg5_full_image_as_row_bands(gpu, reference):
    # BASELINE cfg5 at full size: the 32768^2 u8 image dilated 63x63, computed as 8 virtual row
    # bands (the multi-GPU split on one GPU: each band sees only its rows plus 31-row halos,
    # rmgpu_morph_band_u8), bit-exact against the reference on all host threads
    import torch
    W = H = 32768
    g, nb = 31, 8
    img = torch.empty((H, W), dtype=torch.uint8, device="cuda")
    gpu.generate_device(img, 5)
    out = torch.empty_like(img)
    rows = H // nb
    for k in range(nb):
        r0, r1 = k * rows, (k + 1) * rows
        a, z = max(0, r0 - g), min(H, r1 + g)
        band = img[a:z].clone()  # a separate buffer, as a rank would hold it
        gpu.morph_band_device(band, r0 - a, z - r1, out[r0:r1], 63, 63, DILATE)
        del band
    torch.cuda.synchronize()
    got = to_host(out)
    host = to_host(img)
    del img, out
    torch.cuda.empty_cache()
    want = reference.morph(host, 63, 63, DILATE, nthreads=os.cpu_count() or 8)
    assert np.array_equal(got, want)


def test_cpp_dropin_binary(gpu, tmp_path):
    src = os.path.join(ROOT, "tests", "cpp", "dropin_test.cpp")
    exe = str(tmp_path / "dropin_test")
    pkgdir = os.path.join(ROOT, "paper_2002_09474_b200")
    r = subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), src, "-o", exe,
                        "-L", pkgdir, "-lrectmorph_b200", "-lrmgpu", f"-Wl,-rpath,{pkgdir}"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ALL PASS" in r.stdout


def test_morph_separable_api(gpu, reference, restatement):
    # morph_separable (separable.hpp:44-55, separable.cpp:130-157) with every explicit algorithm /
    # strategy combination -- results never depend on them -- against the reference's own function
    from oracle import LINEAR, VANHERK
    rng = np.random.default_rng(44)
    for c in range(12):
        w, h = int(rng.integers(1, 300)), int(rng.integers(1, 200))
        wx, wy = 2 * int(rng.integers(0, 30)) + 1, 2 * int(rng.integers(0, 30)) + 1
        op = int(rng.integers(0, 2))
        border, bval = int(rng.integers(0, 2)), int(rng.integers(0, 256))
        img = restatement.generate(w, h, 500 + c)
        for ha, va, vs in ((1, 1, 0), (2, 2, 1), (1, 2, 1), (2, 1, 0), (0, 0, 0)):
            want = reference.morph_separable(img, wx, wy, op, border, bval, ha, va, vs)
            got = gpu.morph_separable(img, gpu.OpKind(op), gpu.StructuringElement(wx, wy),
                                      gpu.BorderPolicy(border, bval), gpu.PassAlgorithm(ha), gpu.PassAlgorithm(va),
                                      gpu.VerticalStrategy(vs))
            assert np.array_equal(got, want), (c, w, h, wx, wy, op, ha, va, vs)
    assert LINEAR == 1 and VANHERK == 2


@pytest.mark.parametrize("dtype", [np.uint8, np.uint16])
def test_algorithm_hints_never_change_results(gpu, restatement, dtype):
    # the C-ABI's algo_h / algo_v hints (rmgpu.h): Linear on a long wing runs that axis as the
    # direct sliding window, VanHerk / Auto the planner's kernels -- every combination exact
    import torch
    rng = np.random.default_rng(45 + np.dtype(dtype).itemsize)
    mx = int(np.iinfo(dtype).max)
    es = np.dtype(dtype).itemsize
    L = gpu.lib()
    fn = L.rmgpu_morph_u8 if es == 1 else L.rmgpu_morph_u16
    for c in range(24):
        w, h = int(rng.integers(1, 400)), int(rng.integers(1, 300))
        wx, wy = 2 * int(rng.integers(0, 40)) + 1, 2 * int(rng.integers(0, 40)) + 1
        op = int(rng.integers(0, 5))
        border, bval = int(rng.integers(0, 2)), int(rng.integers(0, mx + 1))
        img = restatement.generate(w, h, 900 + c, dtype=dtype)
        want = restatement.morph(img, wx, wy, op, border, bval)
        pad = (-w) % (16 // es)
        for ah, av in ((1, 1), (1, 2), (2, 1), (2, 2), (1, 0), (0, 1)):
            src = to_device(img, pad)
            dst = empty_device(img.shape, dtype, pad)
            rc = fn(src.data_ptr(), src.stride(0) * es, dst.data_ptr(), dst.stride(0) * es, w, h, wx, wy, op, border,
                    bval, ah, av, None)
            assert rc == 0, L.rmgpu_last_error()
            torch.cuda.synchronize()
            assert np.array_equal(to_host(dst), want), (c, w, h, wx, wy, op, border, ah, av)


def test_calibrate_on_gpu(gpu, tmp_path):
    # calibrate (dispatch.cpp:180-248) on the B200: thresholds from the swept set, marked
    # calibrated; a calibrated config steers the planner and still gives the same pixels
    cfg = gpu.calibrate(512, 384, [3, 5, 7, 9, 15, 31], 3)
    assert cfg.source == "calibrated"
    assert cfg.threshold_h in (1, 3, 5, 7, 9, 15, 31) and cfg.threshold_v in (1, 3, 5, 7, 9, 15, 31)
    img = np.random.default_rng(9).integers(0, 256, (301, 277), dtype=np.uint8)
    for t in (cfg, gpu.DispatchConfig(101, 101, "calibrated"), gpu.DispatchConfig(1, 1, "calibrated")):
        for (wx, wy) in ((31, 15), (9, 63), (3, 3)):
            a = gpu.erode(img, gpu.make_se(wx, wy), gpu.BorderPolicy(), t)
            b = gpu.erode(img, gpu.make_se(wx, wy))
            assert np.array_equal(a, b), (t, wx, wy)
    src = os.path.join(ROOT, "tests", "cpp", "config_test.cpp")
    exe = str(tmp_path / "config_test")
    pkgdir = os.path.join(ROOT, "paper_2002_09474_b200")
    r = subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), src, "-o", exe,
                        "-L", pkgdir, "-lrectmorph_b200", "-lrmgpu", f"-Wl,-rpath,{pkgdir}"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([exe, str(tmp_path), "--gpu"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "config_test ok" in r.stdout


@pytest.mark.parametrize("dtype", [np.uint8, np.uint16])
def test_row_bands_with_overlapped_exchange_one_gpu(gpu, restatement, dtype):
    # the multi-GPU row-band pipeline driven from one process (shard.morph_bands_local): band
    # buffers holding only their own rows, halos copied between them on each band's stream while
    # the interior rows are computed, then the edge rows -- rmgpu_morph_band_* behind a real
    # exchange, against the whole-image oracle
    import torch
    from paper_2002_09474_b200.shard import morph_bands_local
    rng = np.random.default_rng(61 + np.dtype(dtype).itemsize)
    mx = int(np.iinfo(dtype).max)
    for c in range(10):
        w, h = int(rng.integers(16, 900)), int(rng.integers(64, 700))
        gy = int(rng.integers(1, 40))
        nb = int(rng.integers(2, max(3, min(8, h // max(gy, 1)))))
        wx, wy = 2 * int(rng.integers(0, 30)) + 1, 2 * gy + 1
        op = int(rng.integers(0, 2)) if c % 3 else GRADIENT
        border, bval = int(rng.integers(0, 2)), int(rng.integers(0, mx + 1))
        img = restatement.generate(w, h, 1300 + c, dtype=dtype)
        src = to_device(img)
        out = empty_device(img.shape, dtype)
        morph_bands_local(src, out, nb, wx, wy, op, border, bval)
        torch.cuda.synchronize()
        assert np.array_equal(to_host(out), restatement.morph(img, wx, wy, op, border, bval)), \
            (c, w, h, wx, wy, op, border, nb)
