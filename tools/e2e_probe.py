"""Host-entry (e2e) probe: copies alone vs rmgpu_morph_host_u8 with different band counts.
python tools/e2e_probe.py"""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2002_09474_b200 as pkg

n = 4096
h_in = torch.randint(0, 256, (n, n), dtype=torch.uint8).pin_memory()
h_out = torch.empty_like(h_in).pin_memory()
d_a = torch.empty((n, n), dtype=torch.uint8, device="cuda")
d_b = torch.empty_like(d_a)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def copies(kind, reps=20):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        if kind in ("h2d", "both"):
            with torch.cuda.stream(s1):
                d_a.copy_(h_in, non_blocking=True)
        if kind in ("d2h", "both"):
            with torch.cuda.stream(s2):
                h_out.copy_(d_b, non_blocking=True)
        torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / reps
    print(f"copy {kind}: {dt * 1e6:.0f} us per 16 MiB", flush=True)


L = pkg.lib()


def host(w, bands, reps=20):
    pkg.debug_set("host_bands", bands)
    for _ in range(3):
        L.rmgpu_morph_host_u8(C.c_void_p(h_in.data_ptr()), n, C.c_void_p(h_out.data_ptr()), n, n, n, w, w, 0, 0, 0, 0, 0)
    t = time.perf_counter()
    for _ in range(reps):
        L.rmgpu_morph_host_u8(C.c_void_p(h_in.data_ptr()), n, C.c_void_p(h_out.data_ptr()), n, n, n, w, w, 0, 0, 0, 0, 0)
    dt = (time.perf_counter() - t) / reps
    print(f"host {w}x{w} bands={bands}: {dt * 1e6:.0f} us ({n * n / dt / 1e9:.1f} Gpix/s)", flush=True)


for k in ("h2d", "d2h", "both"):
    copies(k)
for w in (3, 63):
    for b in (1, 2, 4, 6, 8, 12, 16, 32):
        host(w, b)
