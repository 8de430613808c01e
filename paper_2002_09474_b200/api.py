"""Python mirror of the reference ``rectmorph`` operator API over the GPU C-ABI.

Names, argument meaning and error behaviour follow the reference's public headers
(/root/reference/proj/core/include/rectmorph/*.hpp) so the parity tests read like the
reference's own tests:

* host level (numpy in, numpy out, value semantics): ``erode``, ``dilate``, ``opening``,
  ``closing``, ``gradient``, ``morph_separable``, ``horizontal_pass``, ``vertical_pass_direct``,
  ``vertical_pass_via_transpose``, ``transpose_image``, ``transpose_tile``,
  ``linear_window_1d``, ``van_herk_1d``, ``resolve``, ``make_se``;
* device level (torch CUDA tensors, stream-ordered, no copies): ``morph_device``,
  ``morph_batched_device``, ``morph_band_device``, ``transpose_device``,
  ``transpose_tiles_device``, ``generate_device``.

Errors raise ``Error`` carrying the reference's ``Errc`` (error.hpp:10-22) or ``GpuError``.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from enum import IntEnum

import numpy as np

from ._native import lib


class Errc(IntEnum):
    ZeroExtent = 0
    EvenExtent = 1
    UnsupportedTile = 2
    BadMagic = 3
    BadHeader = 4
    UnsupportedMaxval = 5
    TruncatedData = 6
    BadConfig = 7
    InsufficientReps = 8
    IoError = 9
    BadArgument = 10


class Error(RuntimeError):
    """rectmorph::Error (error.hpp:24-33)."""

    def __init__(self, code: Errc, message: str):
        super().__init__(message)
        self.code = code


class GpuError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"[{status}] {message}")
        self.status = status


class OpKind(IntEnum):
    Erode = 0
    Dilate = 1


class PassAlgorithm(IntEnum):
    Auto = 0
    Linear = 1
    VanHerk = 2


class VerticalStrategy(IntEnum):
    Direct = 0
    ViaTranspose = 1


class Axis(IntEnum):
    Horizontal = 0
    Vertical = 1


# C-ABI op codes (rmgpu.h)
ERODE, DILATE, OPEN, CLOSE, GRADIENT = 0, 1, 2, 3, 4
REPLICATE, CONSTANT = 0, 1


@dataclass(frozen=True)
class BorderPolicy:
    mode: int = REPLICATE
    value: int = 0

    @staticmethod
    def replicate() -> "BorderPolicy":
        return BorderPolicy(REPLICATE, 0)

    @staticmethod
    def constant(v: int) -> "BorderPolicy":
        return BorderPolicy(CONSTANT, int(v))


@dataclass(frozen=True)
class StructuringElement:
    width: int = 1
    height: int = 1

    @property
    def wing_x(self) -> int:
        return self.width // 2

    @property
    def wing_y(self) -> int:
        return self.height // 2


@dataclass
class DispatchConfig:
    threshold_h: int = 69
    threshold_v: int = 59
    source: str = "paper"


def identity_value(op: OpKind, dtype=np.uint8) -> int:
    return int(np.iinfo(dtype).max) if op == OpKind.Erode else 0


def _check(rc: int) -> None:
    if rc == 0:
        return
    msg = lib().rmgpu_last_error().decode(errors="replace")
    if 1 <= rc <= 11:
        raise Error(Errc(rc - 1), msg)
    raise GpuError(rc, msg or lib().rmgpu_status_string(rc).decode())


def make_se(width: int, height: int) -> StructuringElement:
    """image.cpp:18-24."""
    if width < 1 or height < 1:
        raise Error(Errc.ZeroExtent, "structuring element extents must be >= 1")
    if width % 2 == 0 or height % 2 == 0:
        raise Error(Errc.EvenExtent, "structuring element extents must be odd")
    return StructuringElement(width, height)


def _validate_window(window: int) -> None:
    if window < 1:
        raise Error(Errc.ZeroExtent, "window extent must be >= 1")
    if window % 2 == 0:
        raise Error(Errc.EvenExtent, "window extent must be odd")


def resolve(algo: PassAlgorithm, window: int, axis: Axis, cfg: DispatchConfig | None = None) -> PassAlgorithm:
    cfg = cfg or DispatchConfig()
    return PassAlgorithm(lib().rmgpu_resolve(int(algo), window, int(axis), cfg.threshold_h, cfg.threshold_v))


def format_config(cfg: DispatchConfig) -> str:
    """dispatch.hpp:46-50: "threshold_h=..\\nthreshold_v=..\\nsource=paper|calibrated\\n"."""
    buf = C.create_string_buffer(96)
    n = lib().rmgpu_format_config(cfg.threshold_h, cfg.threshold_v, 1 if cfg.source == "calibrated" else 0,
                                  buf, len(buf))
    return buf.value[:n].decode()


def parse_config(text: str) -> DispatchConfig:
    """Strict inverse of format_config (dispatch.hpp:52-55); Error(Errc.BadConfig) otherwise."""
    th, tv, src = C.c_int(0), C.c_int(0), C.c_int(0)
    _check(lib().rmgpu_parse_config(text.encode(), C.byref(th), C.byref(tv), C.byref(src)))
    return DispatchConfig(th.value, tv.value, "calibrated" if src.value == 1 else "paper")


def load_config(path: str) -> DispatchConfig:
    try:
        with open(path, "rb") as f:
            text = f.read().decode(errors="replace")
    except OSError:
        raise Error(Errc.IoError, f"cannot open config '{path}'") from None
    try:
        return parse_config(text)
    except Error as e:
        raise Error(e.code, f"{path}: {e}") from None


def save_config(path: str, cfg: DispatchConfig) -> None:
    try:
        with open(path, "wb") as f:
            f.write(format_config(cfg).encode())
    except OSError:
        raise Error(Errc.IoError, f"cannot open '{path}' for writing") from None


def calibrate(width: int, height: int, windows, reps: int) -> DispatchConfig:
    """dispatch.hpp:59-66 measured on the current GPU (rmgpu_calibrate)."""
    ws = list(windows)
    arr = (C.c_int * max(1, len(ws)))(*ws)
    th, tv = C.c_int(0), C.c_int(0)
    _check(lib().rmgpu_calibrate(width, height, arr, len(ws), reps, C.byref(th), C.byref(tv)))
    return DispatchConfig(th.value, tv.value, "calibrated")


def _hints(se, cfg: DispatchConfig | None) -> tuple[int, int]:
    """A Calibrated config steers the GPU planner axis by axis; the paper's thresholds do not."""
    if cfg is None or cfg.source != "calibrated":
        return 0, 0
    return (int(resolve(PassAlgorithm.Auto, se.width, Axis.Horizontal, cfg)),
            int(resolve(PassAlgorithm.Auto, se.height, Axis.Vertical, cfg)))


# ------------------------------------------------------------------------------------------
# host level
# ------------------------------------------------------------------------------------------
def _host_image(img: np.ndarray) -> np.ndarray:
    img = np.asarray(img)
    if img.ndim != 2 or img.dtype not in (np.uint8, np.uint16):
        raise Error(Errc.BadArgument, "expected a 2-D uint8 or uint16 image")
    return np.ascontiguousarray(img)


def _morph_host(img: np.ndarray, se: StructuringElement, border: BorderPolicy, op: int,
                hints: tuple[int, int] = (0, 0)) -> np.ndarray:
    img = _host_image(img)
    h, w = img.shape
    out = np.empty_like(img)
    es = img.itemsize
    fn = lib().rmgpu_morph_host_u8 if es == 1 else lib().rmgpu_morph_host_u16
    _check(fn(img.ctypes.data, w * es, out.ctypes.data, w * es, w, h, se.width, se.height, op,
              border.mode, border.value, hints[0], hints[1]))
    return out


def erode(img, se, border=BorderPolicy(), cfg=None):
    return _morph_host(img, se, border, ERODE, _hints(se, cfg))


def dilate(img, se, border=BorderPolicy(), cfg=None):
    return _morph_host(img, se, border, DILATE, _hints(se, cfg))


def opening(img, se, border=BorderPolicy(), cfg=None):
    return _morph_host(img, se, border, OPEN, _hints(se, cfg))


def closing(img, se, border=BorderPolicy(), cfg=None):
    return _morph_host(img, se, border, CLOSE, _hints(se, cfg))


def gradient(img, se, border=BorderPolicy(), cfg=None):
    return _morph_host(img, se, border, GRADIENT, _hints(se, cfg))


def morph_separable(img, op: OpKind, se, border=BorderPolicy(), h_algo=PassAlgorithm.Auto,
                    v_algo=PassAlgorithm.Auto, v_strategy=None):
    _validate_window(se.width)
    _validate_window(se.height)
    # the explicit per-axis algorithms are GPU planner hints (rmgpu.h); v_strategy has no GPU
    # counterpart (both strategies are the same fused column pass)
    return _morph_host(img, se, border, int(op), (int(h_algo), int(v_algo)))


def _pass(which: int, img, op: OpKind, window: int, border: BorderPolicy) -> np.ndarray:
    _validate_window(window)
    img = _host_image(img)
    if img.dtype != np.uint8:
        raise Error(Errc.BadArgument, "pass-level API is 8-bit like the reference")
    h, w = img.shape
    out = np.empty_like(img)
    _check(lib().rmgpu_pass_host_u8(which, img.ctypes.data, w, out.ctypes.data, w, w, h, window, int(op),
                                    border.mode, border.value, 0))
    return out


def horizontal_pass(img, op, window, border=BorderPolicy(), algo=PassAlgorithm.Auto):
    return _pass(0, img, op, window, border)


def vertical_pass_direct(img, op, window, border=BorderPolicy()):
    return _pass(1, img, op, window, border)


def vertical_pass_via_transpose(img, op, window, border=BorderPolicy(), algo=PassAlgorithm.Auto):
    return _pass(2, img, op, window, border)


def transpose_image(img: np.ndarray) -> np.ndarray:
    img = _host_image(img)
    h, w = img.shape
    out = np.empty((w, h), dtype=img.dtype)
    es = img.itemsize
    fn = lib().rmgpu_transpose_host_u8 if es == 1 else lib().rmgpu_transpose_host_u16
    _check(fn(img.ctypes.data, w * es, out.ctypes.data, h * es, w, h))
    return out


def transpose_tile(data: np.ndarray, stride: int, n: int, offset: int = 0) -> None:
    """In-place n x n tile transpose (transpose.hpp:36-38); ``data`` is a flat numpy buffer."""
    if not data.flags.c_contiguous:
        raise Error(Errc.BadArgument, "tile buffer must be contiguous")
    ptr = data.ctypes.data + offset * data.itemsize
    _check(lib().rmgpu_transpose_tiles_host(ptr, data.itemsize, 1, n, stride, 0))


def transpose_tiles(data: np.ndarray, n: int) -> None:
    """In-place transpose of a flat batch of contiguous n x n tiles."""
    if not data.flags.c_contiguous:
        raise Error(Errc.BadArgument, "tile buffer must be contiguous")
    _check(lib().rmgpu_transpose_tiles_host(data.ctypes.data, data.itemsize, data.size // (n * n), n, n, n * n))


@dataclass
class OpCounter:
    comparisons: int = 0

    def reset(self) -> None:
        self.comparisons = 0


def _window_1d(sig, window, op, border, counter, vanherk):
    _validate_window(window)
    sig = np.ascontiguousarray(sig, dtype=np.uint8)
    if counter is not None:
        counter.reset()
    out = np.empty_like(sig)
    n = sig.size
    if n == 0:
        return out
    if window == 1:
        out[:] = sig
        return out
    _check(lib().rmgpu_window_1d_host_u8(sig.ctypes.data, n, window, int(op), border.mode, border.value,
                                         2 if vanherk else 1, out.ctypes.data))
    if counter is not None:  # closed form of the reference algorithm (sliding_extrema.cpp:131,139)
        if vanherk:
            ln = n + window - 1
            counter.comparisons = 2 * (ln - (ln + window - 1) // window) + n
        else:
            counter.comparisons = (window - 1) * n
    return out


def linear_window_1d(sig, window, op, border=BorderPolicy(), counter=None):
    return _window_1d(sig, window, op, border, counter, False)


def van_herk_1d(sig, window, op, border=BorderPolicy(), counter=None):
    return _window_1d(sig, window, op, border, counter, True)


# ------------------------------------------------------------------------------------------
# PGM files (pgm.hpp:10-24): host-side format code, the same rules as the C++ drop-in
# ------------------------------------------------------------------------------------------
_PGM_MAX_SIDE = 1 << 20


def read_pgm(data: bytes) -> np.ndarray:
    """P5 / P2, maxval 255, '#' comments in the header (and between P2 tokens)."""
    pos = 0
    n = len(data)

    def to_token() -> bool:
        nonlocal pos
        while pos < n:
            c = data[pos]
            if c == 0x23:  # '#': to the end of the line
                while pos < n and data[pos] != 0x0A:
                    pos += 1
            elif c in b" \t\n\r\v\f":
                pos += 1
            else:
                return True
        return False

    def token(what: str, at_eof: Errc) -> int:
        nonlocal pos
        if not to_token():
            raise Error(at_eof, f"stream ended before the {what}")
        if not 0x30 <= data[pos] <= 0x39:
            raise Error(Errc.BadHeader, f"the {what} is not a number")
        v = 0
        while pos < n and 0x30 <= data[pos] <= 0x39:
            v = v * 10 + data[pos] - 0x30
            pos += 1
            if v > 100 * _PGM_MAX_SIDE:
                raise Error(Errc.BadHeader, f"the {what} is out of range")
        return v

    if n < 2 or data[0] != 0x50 or data[1] not in (0x35, 0x32):
        raise Error(Errc.BadMagic, "not a P5 / P2 PGM stream")
    binary = data[1] == 0x35
    pos = 2
    w, h = token("width", Errc.BadHeader), token("height", Errc.BadHeader)
    if not (1 <= w <= _PGM_MAX_SIDE and 1 <= h <= _PGM_MAX_SIDE):
        raise Error(Errc.BadHeader, "image extents out of range")
    if token("maxval", Errc.BadHeader) != 255:
        raise Error(Errc.UnsupportedMaxval, "maxval must be 255")
    if binary:
        if pos >= n or data[pos] not in b" \t\n\r\v\f":
            raise Error(Errc.BadHeader, "no whitespace after the maxval")
        pos += 1
        if n - pos < w * h:
            raise Error(Errc.TruncatedData, "pixel data ends early")
        return np.frombuffer(data, np.uint8, w * h, pos).reshape(h, w).copy()
    out = np.empty((h, w), np.uint8)
    for i in range(w * h):
        v = token("pixel", Errc.TruncatedData)
        if v > 255:
            raise Error(Errc.BadHeader, "a pixel exceeds the maxval")
        out.flat[i] = v
    return out


def write_pgm(img: np.ndarray, binary: bool = True) -> bytes:
    img = np.asarray(img)
    if img.ndim != 2 or img.dtype != np.uint8:
        raise Error(Errc.BadArgument, "expected a 2-D uint8 image")
    if img.size == 0:
        raise Error(Errc.BadArgument, "an empty image has no PGM form")
    h, w = img.shape
    head = f"{'P5' if binary else 'P2'}\n{w} {h}\n255\n".encode()
    if binary:
        return head + np.ascontiguousarray(img).tobytes()
    return head + "".join(" ".join(str(int(v)) for v in row) + "\n" for row in img).encode()


def load_pgm(path: str) -> np.ndarray:
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError:
        raise Error(Errc.IoError, f"cannot open '{path}'") from None
    try:
        return read_pgm(data)
    except Error as e:
        raise Error(e.code, f"{path}: {e}") from None


def store_pgm(path: str, img: np.ndarray, binary: bool = True) -> None:
    data = write_pgm(img, binary)
    try:
        with open(path, "wb") as f:
            f.write(data)
    except OSError:
        raise Error(Errc.IoError, f"cannot open '{path}' for writing") from None


# ------------------------------------------------------------------------------------------
# device level (torch CUDA tensors); pitch = tensor.stride(0) * itemsize
# ------------------------------------------------------------------------------------------
def _dev(t):
    import torch
    if not t.is_cuda:
        raise Error(Errc.BadArgument, "expected a CUDA tensor")
    if t.dtype not in (torch.uint8, torch.uint16):
        raise Error(Errc.BadArgument, "expected uint8 or uint16")
    if t.stride(-1) != 1:
        raise Error(Errc.BadArgument, "rows must be contiguous")
    return t


def _same(src, dst, what: str = "dst") -> None:
    """dst must match src in dtype and device (and shape, checked by the callers)."""
    if src.dtype != dst.dtype or src.device != dst.device:
        raise Error(Errc.BadArgument, f"{what} must have the source's dtype and device")


def _stream_ptr(stream):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def morph_device(src, dst, wx: int, wy: int, op: int, border: int = REPLICATE, value: int = 0,
                 stream=None) -> None:
    """2-D tensors [H, W] (row pitch from stride(0)). Asynchronous on ``stream``."""
    _dev(src), _dev(dst)
    _same(src, dst)
    if src.dim() != 2 or tuple(dst.shape) != tuple(src.shape):
        raise Error(Errc.BadArgument, "src and dst must be 2-D tensors of the same shape")
    h, w = src.shape
    es = src.element_size()
    fn = lib().rmgpu_morph_u8 if es == 1 else lib().rmgpu_morph_u16
    _check(fn(src.data_ptr(), src.stride(0) * es, dst.data_ptr(), dst.stride(0) * es, w, h, wx, wy, op,
              border, value, 0, 0, _stream_ptr(stream)))


def morph_batched_device(src, dst, wx, wy, op, border=REPLICATE, value=0, stream=None) -> None:
    """3-D tensors [B, H, W]."""
    _dev(src), _dev(dst)
    _same(src, dst)
    if src.dim() != 3 or tuple(dst.shape) != tuple(src.shape):
        raise Error(Errc.BadArgument, "src and dst must be 3-D tensors of the same shape")
    b, h, w = src.shape
    es = src.element_size()
    fn = lib().rmgpu_morph_batched_u8 if es == 1 else lib().rmgpu_morph_batched_u16
    _check(fn(src.data_ptr(), src.stride(1) * es, src.stride(0) * es, dst.data_ptr(), dst.stride(1) * es,
              dst.stride(0) * es, b, w, h, wx, wy, op, border, value, _stream_ptr(stream)))


def morph_band_device(src_with_halo, rows_above: int, rows_below: int, dst, wx, wy, op, border=REPLICATE,
                      value=0, stream=None) -> None:
    """``src_with_halo`` holds rows_above + band_rows + rows_below rows; dst holds band_rows."""
    _dev(src_with_halo), _dev(dst)
    _same(src_with_halo, dst)
    if src_with_halo.dim() != 2 or dst.dim() != 2 or src_with_halo.shape[1] != dst.shape[1]:
        raise Error(Errc.BadArgument, "src_with_halo and dst must be 2-D tensors of the same width")
    if rows_above < 0 or rows_below < 0 or src_with_halo.shape[0] < rows_above + dst.shape[0] + rows_below:
        raise Error(Errc.BadArgument, "src_with_halo must hold rows_above + band rows + rows_below rows")
    rows, w = dst.shape
    es = dst.element_size()
    base = src_with_halo.data_ptr() + rows_above * src_with_halo.stride(0) * es
    fn = lib().rmgpu_morph_band_u8 if es == 1 else lib().rmgpu_morph_band_u16
    _check(fn(base, src_with_halo.stride(0) * es, dst.data_ptr(), dst.stride(0) * es, w, rows, rows_above,
              rows_below, wx, wy, op, border, value, _stream_ptr(stream)))


def transpose_device(src, dst, stream=None) -> None:
    _dev(src), _dev(dst)
    _same(src, dst)
    if src.dim() != 2 or tuple(dst.shape) != (src.shape[1], src.shape[0]):
        raise Error(Errc.BadArgument, "dst must be the W x H transpose shape of src")
    h, w = src.shape
    es = src.element_size()
    fn = lib().rmgpu_transpose_u8 if es == 1 else lib().rmgpu_transpose_u16
    _check(fn(src.data_ptr(), src.stride(0) * es, dst.data_ptr(), dst.stride(0) * es, w, h, _stream_ptr(stream)))


def transpose_tiles_device(data, n: int, n_tiles: int | None = None, row_stride: int | None = None,
                           tile_step: int | None = None, stream=None) -> None:
    import torch
    es = data.element_size()
    n_tiles = data.numel() // (n * n) if n_tiles is None else n_tiles
    fn = {1: lib().rmgpu_transpose_tiles_u8, 2: lib().rmgpu_transpose_tiles_u16,
          4: lib().rmgpu_transpose_tiles_u32}[es]
    _check(fn(data.data_ptr(), n_tiles, n, n if row_stride is None else row_stride,
              n * n if tile_step is None else tile_step, _stream_ptr(stream)))


def generate_device(dst, seed: int, stream_id: int = 0, stream=None) -> None:
    _dev(dst)
    h, w = dst.shape
    es = dst.element_size()
    fn = lib().rmgpu_generate_u8 if es == 1 else lib().rmgpu_generate_u16
    _check(fn(dst.data_ptr(), dst.stride(0) * es, w, h, seed, stream_id, _stream_ptr(stream)))


def launch_count() -> int:
    return int(lib().rmgpu_launch_count())


def debug_set(knob: str, value: int) -> None:
    """Override a planner tuning knob (rmgpu_debug_set); value < 0 removes the override. Knobs
    choose kernel variants / launch geometry only, never results."""
    lib().rmgpu_debug_set(knob.encode(), int(value))


def plan_name(elem_bytes: int, w: int, h: int, wx: int, wy: int, op: int = ERODE) -> str:
    return lib().rmgpu_plan_name(elem_bytes, w, h, wx, wy, op).decode()
