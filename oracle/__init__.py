"""TEST INFRASTRUCTURE ONLY -- CPU checkers for the CUDA path.

Two checkers, both loaded through ctypes:

* ``restatement()``: ``oracle/liboracle.so``, the plain-C restatement of the
  reference algorithms in ``oracle/rmoracle.c`` (u8 and the u16 extension).
* ``reference()``: ``oracle/_ref/librmref.so``, the UNMODIFIED reference core
  (``/root/reference/proj/core/src``) compiled by ``oracle/Makefile`` together
  with ``oracle/ref_shim.cpp``. Absent when the reference was never mounted.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline and
``--impl reference``) may import this package. The product package
``paper_2002_09474_b200`` never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "librmref.so")

ERODE, DILATE, OPEN, CLOSE, GRADIENT = 0, 1, 2, 3, 4
REPLICATE, CONSTANT = 0, 1
LINEAR, VANHERK = 1, 2

_P = C.c_void_p
_S = C.c_size_t
_I = C.c_int
_U = C.c_uint


def build(quiet: bool = True) -> None:
    """Build liboracle.so (and _ref/librmref.so when the reference is mounted)."""
    out = subprocess.run(["make", "-C", HERE], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


class CheckerError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"{what} returned status {code}")
        self.code = code


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


class Restatement:
    """ctypes view of oracle/liboracle.so (rmoracle.h)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        self.lib = C.CDLL(path)
        L = self.lib
        for sfx in ("u8", "u16"):
            f = getattr(L, f"orc_morph_reference_{sfx}")
            f.argtypes = [_P, _S, _I, _I, _P, _S, _I, _I, _I, _I, _U]
            f = getattr(L, f"orc_morph_{sfx}")
            f.argtypes = [_P, _S, _I, _I, _P, _S, _I, _I, _I, _I, _U, _I, _I]
            f = getattr(L, f"orc_transpose_image_{sfx}")
            f.argtypes = [_P, _S, _I, _I, _P, _S]
            f = getattr(L, f"orc_transpose_tile_{sfx}")
            f.argtypes = [_P, _S, _I]
            f = getattr(L, f"orc_transpose_tiles_{sfx}")
            f.argtypes = [_P, _S, _I]
            f = getattr(L, f"orc_generate_{sfx}")
            f.argtypes = [_P, _S, _I, _I, C.c_uint64, C.c_uint64]
            f.restype = None
        L.orc_transpose_tile_u32.argtypes = [_P, _S, _I]
        L.orc_window_1d_u8.argtypes = [_P, _S, _I, _I, _I, _U, _I, _P, C.POINTER(C.c_uint64)]
        L.orc_splitmix64.argtypes = [C.c_uint64]
        L.orc_splitmix64.restype = C.c_uint64

    @staticmethod
    def _sfx(a: np.ndarray) -> str:
        if a.dtype == np.uint8:
            return "u8"
        if a.dtype == np.uint16:
            return "u16"
        raise TypeError(a.dtype)

    def _check(self, rc: int, what: str) -> None:
        if rc != 0:
            raise CheckerError(rc, what)

    def morph(self, src: np.ndarray, wx: int, wy: int, op: int = ERODE, border: int = REPLICATE,
              bval: int = 0, h_algo: int = LINEAR, v_algo: int = LINEAR) -> np.ndarray:
        src = np.ascontiguousarray(src)
        h, w = src.shape
        dst = np.zeros_like(src)
        fn = getattr(self.lib, f"orc_morph_{self._sfx(src)}")
        self._check(fn(_ptr(src), w, w, h, _ptr(dst), w, wx, wy, op, border, bval, h_algo, v_algo),
                    "orc_morph")
        return dst

    def morph_reference(self, src: np.ndarray, wx: int, wy: int, op: int = ERODE,
                        border: int = REPLICATE, bval: int = 0) -> np.ndarray:
        src = np.ascontiguousarray(src)
        h, w = src.shape
        dst = np.zeros_like(src)
        fn = getattr(self.lib, f"orc_morph_reference_{self._sfx(src)}")
        self._check(fn(_ptr(src), w, w, h, _ptr(dst), w, wx, wy, op, border, bval),
                    "orc_morph_reference")
        return dst

    def transpose_image(self, src: np.ndarray) -> np.ndarray:
        src = np.ascontiguousarray(src)
        h, w = src.shape
        dst = np.zeros((w, h), dtype=src.dtype)
        fn = getattr(self.lib, f"orc_transpose_image_{self._sfx(src)}")
        self._check(fn(_ptr(src), w, w, h, _ptr(dst), h), "orc_transpose_image")
        return dst

    def transpose_tiles(self, tiles: np.ndarray, n: int) -> np.ndarray:
        """Transposes a flat array of contiguous n x n tiles (copy returned)."""
        t = np.ascontiguousarray(tiles).copy()
        n_tiles = t.size // (n * n)
        fn = getattr(self.lib, f"orc_transpose_tiles_{self._sfx(t)}")
        self._check(fn(_ptr(t), n_tiles, n), "orc_transpose_tiles")
        return t

    def transpose_tile(self, data: np.ndarray, stride: int, n: int) -> None:
        """In place, like rectmorph::transpose_tile (transpose.hpp:36-38)."""
        if data.dtype == np.uint32:
            rc = self.lib.orc_transpose_tile_u32(_ptr(data), stride, n)
        else:
            rc = getattr(self.lib, f"orc_transpose_tile_{self._sfx(data)}")(_ptr(data), stride, n)
        self._check(rc, "orc_transpose_tile")

    def window_1d(self, sig: np.ndarray, window: int, op: int = ERODE, border: int = REPLICATE,
                  bval: int = 0, algo: int = LINEAR):
        sig = np.ascontiguousarray(sig, dtype=np.uint8)
        out = np.zeros_like(sig)
        cnt = C.c_uint64(0)
        self._check(self.lib.orc_window_1d_u8(_ptr(sig), sig.size, window, op, border, bval, algo,
                                              _ptr(out), C.byref(cnt)), "orc_window_1d_u8")
        return out, cnt.value

    def generate(self, w: int, h: int, seed: int, stream: int = 0, dtype=np.uint8) -> np.ndarray:
        dst = np.zeros((h, w), dtype=dtype)
        fn = getattr(self.lib, f"orc_generate_{self._sfx(dst)}")
        fn(_ptr(dst), w, w, h, seed, stream)
        return dst


class Reference:
    """ctypes view of oracle/_ref/librmref.so: the reference's own code."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = C.CDLL(path)
        L = self.lib
        L.rmref_morph_u8.argtypes = [_P, _S, _I, _I, _P, _S, _I, _I, _I, _I, _U, _I, _I, _I]
        L.rmref_morph_separable_u8.argtypes = [_P, _S, _I, _I, _P, _S, _I, _I, _I, _I, _U, _I, _I,
                                               _I]
        L.rmref_morph_reference_u8.argtypes = [_P, _S, _I, _I, _P, _S, _I, _I, _I, _I, _U]
        L.rmref_pass_u8.argtypes = [_I, _P, _S, _I, _I, _P, _S, _I, _I, _I, _U, _I]
        L.rmref_window_1d_u8.argtypes = [_I, _P, _S, _I, _I, _I, _U, _P, C.POINTER(C.c_uint64)]
        L.rmref_transpose_image_u8.argtypes = [_P, _S, _I, _I, _P, _S, _I]
        L.rmref_transpose_tile_u8.argtypes = [_P, _S, _I]
        L.rmref_transpose_tile_u16.argtypes = [_P, _S, _I]
        L.rmref_transpose_tile_u32.argtypes = [_P, _S, _I]
        L.rmref_transpose_tiles_u8.argtypes = [_P, _S, _I, _I]
        L.rmref_transpose_tiles_u16.argtypes = [_P, _S, _I, _I]
        L.rmref_calibrate.argtypes = [_I, _I, C.POINTER(C.c_int), _I, _I, C.POINTER(C.c_int),
                                      C.POINTER(C.c_int)]
        L.rmref_set_pinning.argtypes = [_I]
        L.rmref_set_pinning.restype = None

    @staticmethod
    def available(path: str = REF_SO) -> bool:
        return os.path.exists(path)

    def _check(self, rc: int, what: str) -> None:
        if rc != 0:
            raise CheckerError(rc, what)

    def morph(self, src: np.ndarray, wx: int, wy: int, op: int = ERODE, border: int = REPLICATE,
              bval: int = 0, threshold_h: int = 69, threshold_v: int = 59, nthreads: int = 1,
              out: np.ndarray | None = None) -> np.ndarray:
        """rectmorph::{erode,dilate,opening,closing,gradient} (dispatch.cpp:38-71)."""
        assert src.dtype == np.uint8
        src = np.ascontiguousarray(src)
        h, w = src.shape
        dst = np.empty_like(src) if out is None else out
        self._check(self.lib.rmref_morph_u8(_ptr(src), w, w, h, _ptr(dst), w, wx, wy, op, border,
                                            bval, threshold_h, threshold_v, nthreads),
                    "rmref_morph_u8")
        return dst

    def morph_separable(self, src, wx, wy, op, border, bval, h_algo, v_algo, v_strategy):
        src = np.ascontiguousarray(src, dtype=np.uint8)
        h, w = src.shape
        dst = np.empty_like(src)
        self._check(self.lib.rmref_morph_separable_u8(_ptr(src), w, w, h, _ptr(dst), w, wx, wy, op,
                                                      border, bval, h_algo, v_algo, v_strategy),
                    "rmref_morph_separable_u8")
        return dst

    def morph_reference(self, src, wx, wy, op=ERODE, border=REPLICATE, bval=0):
        src = np.ascontiguousarray(src, dtype=np.uint8)
        h, w = src.shape
        dst = np.empty_like(src)
        self._check(self.lib.rmref_morph_reference_u8(_ptr(src), w, w, h, _ptr(dst), w, wx, wy, op,
                                                      border, bval), "rmref_morph_reference_u8")
        return dst

    def pass_(self, which: int, src, window, op=ERODE, border=REPLICATE, bval=0, algo=0):
        """which: 0 horizontal_pass, 1 vertical_pass_direct, 2 vertical_pass_via_transpose."""
        src = np.ascontiguousarray(src, dtype=np.uint8)
        h, w = src.shape
        dst = np.empty_like(src)
        self._check(self.lib.rmref_pass_u8(which, _ptr(src), w, w, h, _ptr(dst), w, window, op,
                                           border, bval, algo), "rmref_pass_u8")
        return dst

    def window_1d(self, sig, window, op=ERODE, border=REPLICATE, bval=0, algo=LINEAR):
        sig = np.ascontiguousarray(sig, dtype=np.uint8)
        out = np.zeros_like(sig)
        cnt = C.c_uint64(0)
        self._check(self.lib.rmref_window_1d_u8(algo, _ptr(sig), sig.size, window, op, border, bval,
                                                _ptr(out), C.byref(cnt)), "rmref_window_1d_u8")
        return out, cnt.value

    def transpose_image(self, src: np.ndarray, nthreads: int = 1,
                        out: np.ndarray | None = None) -> np.ndarray:
        src = np.ascontiguousarray(src, dtype=np.uint8)
        h, w = src.shape
        dst = np.empty((w, h), dtype=np.uint8) if out is None else out
        self._check(self.lib.rmref_transpose_image_u8(_ptr(src), w, w, h, _ptr(dst), h, nthreads),
                    "rmref_transpose_image_u8")
        return dst

    def transpose_tile(self, data: np.ndarray, stride: int, n: int) -> None:
        fn = {np.dtype(np.uint8): self.lib.rmref_transpose_tile_u8,
              np.dtype(np.uint16): self.lib.rmref_transpose_tile_u16,
              np.dtype(np.uint32): self.lib.rmref_transpose_tile_u32}[data.dtype]
        self._check(fn(_ptr(data), stride, n), "rmref_transpose_tile")

    def transpose_tiles(self, tiles: np.ndarray, n: int, nthreads: int = 1,
                        inplace: bool = False) -> np.ndarray:
        t = tiles if inplace else np.ascontiguousarray(tiles).copy()
        fn = self.lib.rmref_transpose_tiles_u8 if t.dtype == np.uint8 else \
            self.lib.rmref_transpose_tiles_u16
        self._check(fn(_ptr(t), t.size // (n * n), n, nthreads), "rmref_transpose_tiles")
        return t

    def set_pinning(self, on: bool) -> None:
        """Pin band worker t to host CPU t (bench.py's timed CPU baseline)."""
        self.lib.rmref_set_pinning(1 if on else 0)

    def calibrate(self, w, h, windows, reps):
        arr = (C.c_int * len(windows))(*windows)
        th, tv = C.c_int(0), C.c_int(0)
        self._check(self.lib.rmref_calibrate(w, h, arr, len(windows), reps, C.byref(th),
                                             C.byref(tv)), "rmref_calibrate")
        return th.value, tv.value


_restatement = None
_reference = None


def restatement() -> Restatement:
    global _restatement
    if _restatement is None:
        _restatement = Restatement()
    return _restatement


def reference() -> Reference:
    global _reference
    if _reference is None:
        _reference = Reference()
    return _reference


# --- numpy restatement of the input generator ----------------------------------
_M64 = (1 << 64) - 1


def splitmix64_np(z: np.ndarray) -> np.ndarray:
    z = (z + np.uint64(0x9E3779B97F4A7C15)).astype(np.uint64)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))
