"""Host-entry (e2e) probe: rmgpu_morph_host_u8 at 4096^2 with different band counts / tapering.
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
L = pkg.lib()


def host(w, bands, taper, reps=20):
    pkg.debug_set("host_bands", bands)
    pkg.debug_set("host_taper", taper)
    for _ in range(3):
        L.rmgpu_morph_host_u8(C.c_void_p(h_in.data_ptr()), n, C.c_void_p(h_out.data_ptr()), n, n, n, w, w, 0, 0, 0, 0, 0)
    t = time.perf_counter()
    for _ in range(reps):
        L.rmgpu_morph_host_u8(C.c_void_p(h_in.data_ptr()), n, C.c_void_p(h_out.data_ptr()), n, n, n, w, w, 0, 0, 0, 0, 0)
    dt = (time.perf_counter() - t) / reps
    print(f"host {w}x{w} bands={bands} taper={taper}: {dt * 1e6:.0f} us ({n * n / dt / 1e9:.1f} Gpix/s)", flush=True)


for w in (3, 63):
    for b in (2, 3, 4, 5, 6, 8):
        for t in (0, 1):
            host(w, b, t)
