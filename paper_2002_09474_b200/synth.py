"""Seeded synthetic inputs for the BASELINE configs, host side.

The same counter-based generator runs on the device (rmgpu_generate_*); both produce identical
bytes, so multi-GPU ranks generate on device while checkers regenerate on the host.

  word(seed, stream, k) = splitmix64(seed * 0xD1B54A32D192ED03 ^ (stream << 40) ^ k)
  u8 pixel i  = byte (i & 7) of word(seed, stream, i >> 3)      (row-major i over W x H)
  u16 pixel i = half (i & 3) of word(seed, stream, i >> 2)

BASELINE names no public dataset; these seeded images stand in with the configs' shapes and value
distributions.
"""
from __future__ import annotations

import numpy as np

_C = 0xD1B54A32D192ED03
_M = (1 << 64) - 1


def splitmix64(z: int) -> int:
    z = (z + 0x9E3779B97F4A7C15) & _M
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M
    return z ^ (z >> 31)


def word(seed: int, stream: int, k: int) -> int:
    return splitmix64((((seed * _C) & _M) ^ (stream << 40) ^ k) & _M)


def _words(seed: int, stream: int, n: int) -> np.ndarray:
    with np.errstate(over="ignore"):
        k = np.arange(n, dtype=np.uint64)
        z = np.uint64((seed * _C) & _M) ^ np.uint64(stream << 40) ^ k
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def generate(w: int, h: int, seed: int, stream: int = 0, dtype=np.uint8) -> np.ndarray:
    per = 8 // np.dtype(dtype).itemsize
    n = w * h
    words = _words(seed, stream, (n + per - 1) // per)
    flat = words.view(dtype)[:n]  # little-endian: byte/half (i % per) of word i // per
    return flat.reshape(h, w).copy()


CFG2_WINDOWS = [(3, 3), (7, 7), (15, 15), (31, 31), (63, 63), (101, 101), (31, 1), (1, 31)]


def cfg2_image(size: int = 4096, seed: int = 2, n_rects: int = 400) -> np.ndarray:
    """BASELINE cfg2: top half uniform random, bottom half a 0/255 mask of n_rects filled
    rectangles of side 5-200 (the "half/half" reading of SURVEY.md 8d)."""
    half = size // 2
    img = np.zeros((size, size), np.uint8)
    img[:half] = generate(size, half, seed, 0)
    for r in range(n_rects):
        u = word(seed, 1, r)
        rw = 5 + (u & 0xFFFF) % 196
        rh = 5 + ((u >> 16) & 0xFFFF) % 196
        x0 = ((u >> 32) & 0xFFFF) % size
        y0 = half + ((u >> 48) & 0xFFFF) % half
        img[y0:min(size, y0 + rh), x0:min(size, x0 + rw)] = 255
    return img
