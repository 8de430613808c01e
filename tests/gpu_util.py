"""Helpers for the GPU parity tests: numpy <-> pitched CUDA tensors without relying on torch's
uint16 arithmetic support (buffers travel as bytes and are re-viewed)."""
from __future__ import annotations

import numpy as np


def to_device(img: np.ndarray, pad_elems: int = 0, poison: int | None = None):
    """Upload a 2-D (or 3-D batch) image into a pitched CUDA tensor; returns the [.., H, W] view."""
    import torch
    img = np.ascontiguousarray(img)
    es = img.itemsize
    *lead, h, w = img.shape
    pitch = w + pad_elems
    full = np.zeros((*lead, h, pitch), dtype=img.dtype)
    if poison is not None:
        full[...] = poison
    full[..., :w] = img
    t = torch.from_numpy(full.view(np.uint8)).cuda()
    if es == 2:
        t = t.view(torch.uint16)
    return t[..., :w]


def empty_device(shape, dtype, pad_elems: int = 0, poison: int = 0):
    """A pitched CUDA buffer whose every byte (padding included) holds `poison`."""
    *lead, h, w = shape
    host = np.full((*lead, h, w), poison, dtype=dtype)
    return to_device(host, pad_elems, poison)


def to_host(t) -> np.ndarray:
    import torch
    es = t.element_size()
    base = t
    if es == 2:
        full = t.contiguous().view(torch.uint8).cpu().numpy().view(np.uint16)
        return full
    return base.contiguous().cpu().numpy()


def to_host_full(t, full_width: int) -> np.ndarray:
    """The whole pitched buffer (including padding) behind a view created by to_device/empty_device."""
    import torch
    es = t.element_size()
    *lead, h, w = t.shape
    storage = torch.as_strided(t, (*lead, h, full_width), t.stride())
    if es == 2:
        return storage.contiguous().view(torch.uint8).cpu().numpy().view(np.uint16)
    return storage.contiguous().cpu().numpy()
