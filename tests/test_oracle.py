"""CPU suite: pins the oracle (the parity checker) before any GPU result is trusted.

1. The restatement (oracle/liboracle.so) reproduces the known-answer vectors in the reference's
   own unit tests (cited per case).
2. It equals the committed golden fixtures made by the reference itself (tests/golden/ref_u8.npz)
   and, for u16, the OpenCV-pinned fixtures (tests/golden/u16.npz).
3. Where the compiled reference (oracle/_ref) is present, it agrees with the restatement on
   randomized cases mirroring acceptance criteria 1-3 and 5 (tests/acceptance.cpp:49-271),
   including constant borders of any value (the reference's brute-force route,
   separable.cpp:137-139) and the multi-threaded band split used as the CPU baseline.
"""
import json
import os

import numpy as np
import pytest

import oracle
from oracle import CLOSE, CONSTANT, DILATE, ERODE, GRADIENT, LINEAR, OPEN, REPLICATE, VANHERK

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ---- 1. known answers from the reference's tests ----------------------------------------------
def test_ramp_3x3_erode(restatement):
    # test_reference.cpp:34-41 / test_separable.cpp:127-138 / fixture_3x3*.pgm (test_cli.cpp:109-120)
    img = np.array([[9, 8, 7], [6, 5, 4], [3, 2, 1]], np.uint8)
    want = np.array([[5, 4, 4], [2, 1, 1], [2, 1, 1]], np.uint8)
    for ha in (LINEAR, VANHERK):
        for va in (LINEAR, VANHERK):
            assert np.array_equal(restatement.morph(img, 3, 3, ERODE, h_algo=ha, v_algo=va), want)
    assert np.array_equal(restatement.morph_reference(img, 3, 3, ERODE), want)


def test_1d_known_answers(restatement):
    # test_sliding_extrema.cpp:18-28; also as a 1x8 row and an 8x1 column (test_separable.cpp:39-50)
    sig = np.array([4, 2, 6, 1, 3, 5, 0, 7], np.uint8)
    er = np.array([2, 2, 1, 1, 1, 0, 0, 0], np.uint8)
    di = np.array([4, 6, 6, 6, 5, 5, 7, 7], np.uint8)
    for algo in (LINEAR, VANHERK):
        assert np.array_equal(restatement.window_1d(sig, 3, ERODE, algo=algo)[0], er)
        assert np.array_equal(restatement.window_1d(sig, 3, DILATE, algo=algo)[0], di)
    assert np.array_equal(restatement.morph(sig[None, :], 3, 1, ERODE)[0], er)
    assert np.array_equal(restatement.morph(sig[:, None], 1, 3, DILATE)[:, 0], di)


def test_constant_border_known_answers(restatement):
    # test_reference.cpp:43-55: 2x2 of 128, 3x3 SE
    img = np.full((2, 2), 128, np.uint8)
    assert np.all(restatement.morph(img, 3, 3, ERODE, CONSTANT, 5) == 5)
    assert np.all(restatement.morph(img, 3, 3, DILATE, CONSTANT, 200) == 200)
    assert np.all(restatement.morph_reference(img, 3, 3, ERODE, CONSTANT, 5) == 5)
    # identity constant = global extremum for a window covering the image (test_reference.cpp:57-76)
    rnd = restatement.generate(7, 5, 3)
    out = restatement.morph(rnd, 15, 11, ERODE, CONSTANT, 255)
    assert np.all(out == rnd.min())


def test_pad_row_semantics(restatement):
    # test_sliding_extrema.cpp:114-124 via the observable 1-D result: {10,20,30}, wing 2
    sig = np.array([10, 20, 30], np.uint8)
    # replicate pad -> {10,10,10,20,30,30,30}; window 5 dilation = {30,30,30}, erosion = {10,10,10}
    assert restatement.window_1d(sig, 5, ERODE)[0].tolist() == [10, 10, 10]
    # constant 9 pad -> {9,9,10,20,30,9,9}: erosion over 5 = {9,9,9}; dilation = {30,30,30}
    assert restatement.window_1d(sig, 5, ERODE, CONSTANT, 9)[0].tolist() == [9, 9, 9]
    assert restatement.window_1d(sig, 3, ERODE, CONSTANT, 9)[0].tolist() == [9, 10, 9]


def test_transpose_known_answers(restatement):
    # test_transpose.cpp:127-133: 3x2 -> 2x3 {1,4,2,5,3,6}
    img = np.array([[1, 2, 3], [4, 5, 6]], np.uint8)
    assert restatement.transpose_image(img).ravel().tolist() == [1, 4, 2, 5, 3, 6]
    # test_transpose.cpp:77-84: 8x8 u16 ramp 8i+j -> 8j+i
    t = np.arange(64, dtype=np.uint16)
    restatement.transpose_tile(t, 8, 8)
    assert np.array_equal(t.reshape(8, 8), np.arange(64, dtype=np.uint16).reshape(8, 8).T)
    # stride wider than the tile leaves neighbours untouched (test_transpose.cpp:86-108)
    buf = np.arange(4 * 10, dtype=np.uint8)
    before = buf.copy()
    restatement.transpose_tile(buf, 10, 4)
    m = before.reshape(4, 10)
    got = buf.reshape(4, 10)
    assert np.array_equal(got[:, :4], m[:, :4].T)
    assert np.array_equal(got[:, 4:], m[:, 4:])
    with pytest.raises(oracle.CheckerError) as e:
        restatement.transpose_tile(buf, 10, 5)
    assert e.value.code == 3  # Errc::UnsupportedTile + 1


def test_window_validation(restatement):
    img = np.zeros((3, 3), np.uint8)
    with pytest.raises(oracle.CheckerError) as e:
        restatement.morph(img, 2, 3)
    assert e.value.code == 2
    with pytest.raises(oracle.CheckerError) as e:
        restatement.morph(img, 0, 3)
    assert e.value.code == 1


def test_generator_pinned(restatement):
    g = json.load(open(os.path.join(GOLDEN, "golden.json")))["generator"]
    assert restatement.generate(64, 1, 7)[0].tolist() == g["u8_seed7_64"]
    assert restatement.generate(16, 1, 9, stream=3, dtype=np.uint16)[0].tolist() == g["u16_seed9_stream3_16"]
    # formula check: pixel i = byte (i&7) of splitmix64(seed*C ^ stream<<40 ^ i>>3)
    L = restatement.lib
    seed, stream = 7, 0
    row = restatement.generate(16, 1, seed, stream)[0]
    for i in range(16):
        w = L.orc_splitmix64(((seed * 0xD1B54A32D192ED03) & ((1 << 64) - 1)) ^ (stream << 40) ^ (i >> 3))
        assert row[i] == (w >> (8 * (i & 7))) & 0xFF


# ---- 2. golden fixtures made by the reference ---------------------------------------------------
def test_golden_u8_from_reference(restatement):
    meta = json.load(open(os.path.join(GOLDEN, "golden.json")))["u8"]
    z = np.load(os.path.join(GOLDEN, "ref_u8.npz"))
    for c in meta["morph"]:
        img = z[f"in{c['case']}"]
        assert np.array_equal(img, restatement.generate(c["w"], c["h"], c["seed"]))
        got = restatement.morph(img, c["wx"], c["wy"], c["op"], c["border"], c["bval"])
        assert np.array_equal(got, z[f"out{c['case']}"]), c
    for j in range(4):
        assert np.array_equal(restatement.transpose_image(z[f"tin{j}"]), z[f"tout{j}"])
    for n in (4, 8, 16):
        for dt in ("uint8", "uint16", "uint32"):
            t = z[f"tile_in_{n}_{dt}"].copy()
            for i in range(3):
                restatement.transpose_tile(t[i * n * n:(i + 1) * n * n], n, n)
            assert np.array_equal(t, z[f"tile_out_{n}_{dt}"])
    for d in meta["one_d"]:
        out, cnt = restatement.window_1d(z[f"d1in_{d['j']}"], d["w"], d["op"], algo=d["algo"])
        assert np.array_equal(out, z[f"d1_{d['j']}_{d['algo']}_{d['op']}"])
        assert cnt == d["comparisons"]


def test_golden_u16(restatement):
    meta = json.load(open(os.path.join(GOLDEN, "golden.json")))["u16"]
    z = np.load(os.path.join(GOLDEN, "u16.npz"))
    for c in meta["morph"]:
        img = z[f"in{c['case']}"]
        got = restatement.morph(img, c["wx"], c["wy"], c["op"], c["border"], c["bval"])
        assert np.array_equal(got, z[f"out{c['case']}"]), c


def test_u16_restatement_properties(restatement):
    # duality with 65535 - v, ordering, idempotence of opening (acceptance.cpp:275-325 at u16)
    a = restatement.generate(37, 29, 77, dtype=np.uint16)
    e = restatement.morph(a, 5, 7, ERODE)
    d = restatement.morph(a, 5, 7, DILATE)
    assert np.array_equal(d, 65535 - restatement.morph(65535 - a, 5, 7, ERODE))
    assert np.all(e <= a) and np.all(a <= d)
    o = restatement.morph(a, 5, 7, OPEN)
    assert np.array_equal(restatement.morph(o, 5, 7, OPEN), o)
    assert np.array_equal(restatement.morph(a, 5, 7, GRADIENT), d - e)


# ---- 3. restatement == reference code on randomized cases --------------------------------------
def test_exhaustive_small_vs_reference(restatement, reference):
    # acceptance criterion 1 shape (acceptance.cpp:49-93), thinned: sizes 1..12, SE <= 9x9
    rng = np.random.default_rng(1)
    for w in range(1, 13):
        for h in range(1, 13, 3):
            img = restatement.generate(w, h, w * 64 + h)
            for sw in range(1, 10, 2):
                sh = int(2 * rng.integers(0, 5) + 1)
                for op in (ERODE, DILATE):
                    for border, bval in ((REPLICATE, 0), (CONSTANT, 255 if op == ERODE else 0)):
                        ref = reference.morph_reference(img, sw, sh, op, border, bval)
                        assert np.array_equal(restatement.morph(img, sw, sh, op, border, bval), ref)
                        for ha in (1, 2):
                            for va in (1, 2):
                                for vs in (0, 1):
                                    got = reference.morph_separable(img, sw, sh, op, border, bval, ha, va, vs)
                                    assert np.array_equal(got, ref)


def test_random_medium_vs_reference(restatement, reference):
    # acceptance criterion 2 shape (acceptance.cpp:97-132) + every op and non-identity constants
    rng = np.random.default_rng(20260815)
    for c in range(120):
        w, h = (int(v) for v in rng.integers(1, 129, 2))
        wx, wy = (int(2 * v + 1) for v in rng.integers(0, 32, 2))
        op = int(rng.integers(0, 5))
        border = int(rng.integers(0, 2))
        bval = int(rng.integers(0, 256))
        img = restatement.generate(w, h, 7000 + c)
        cfg = [(69, 59), (1, 1), (127, 127)][c % 3]
        want = reference.morph(img, wx, wy, op, border, bval, *cfg)
        assert np.array_equal(restatement.morph(img, wx, wy, op, border, bval,
                                                h_algo=1 + c % 2, v_algo=1 + (c // 2) % 2), want), (c, w, h, wx, wy, op)


def test_one_d_vs_reference(restatement, reference):
    # acceptance criteria 3-4 (acceptance.cpp:136-194)
    for n in (1, 2, 7, 33, 64):
        for seed in range(2):
            sig = restatement.generate(n, 1, 100 * n + seed)[0]
            for w in (1, 3, 5, 31, 129):
                for op in (ERODE, DILATE):
                    for border, bval in ((REPLICATE, 0), (CONSTANT, (seed * 31 + n) & 255)):
                        for algo in (LINEAR, VANHERK):
                            a = restatement.window_1d(sig, w, op, border, bval, algo)
                            b = reference.window_1d(sig, w, op, border, bval, algo)
                            assert np.array_equal(a[0], b[0]) and a[1] == b[1]


def test_transpose_vs_reference(restatement, reference):
    # acceptance criterion 5 (acceptance.cpp:238-271)
    for w in range(1, 21, 3):
        for h in range(1, 21, 2):
            img = restatement.generate(w, h, 5000 + w * 32 + h)
            assert np.array_equal(restatement.transpose_image(img), reference.transpose_image(img))
    big = restatement.generate(333, 257, 12)
    assert np.array_equal(reference.transpose_image(big, nthreads=4), big.T)
    for n in (4, 8, 16):
        t = restatement.generate(n * n * 5, 1, n)[0]
        assert np.array_equal(restatement.transpose_tiles(t, n), reference.transpose_tiles(t, n, nthreads=3))


def test_threaded_band_split_is_exact(restatement, reference):
    img = restatement.generate(300, 211, 99)
    for op in (ERODE, DILATE, OPEN, CLOSE, GRADIENT):
        one = reference.morph(img, 9, 13, op, nthreads=1)
        assert np.array_equal(reference.morph(img, 9, 13, op, nthreads=7), one)
        assert np.array_equal(restatement.morph(img, 9, 13, op), one)
