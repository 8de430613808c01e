"""Copy-engine probe: one H2D stream vs several concurrent H2D streams (and the same for D2H), pinned 16 MiB."""
import time
import torch
n = 16 << 20
h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
streams = [torch.cuda.Stream() for _ in range(8)]
def run(kind, k, reps=20):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        part = n // k
        for i in range(k):
            with torch.cuda.stream(streams[i]):
                if kind in ("h2d", "both"):
                    d_a[i * part:(i + 1) * part].copy_(h_in[i * part:(i + 1) * part], non_blocking=True)
            with torch.cuda.stream(streams[k + i if k + i < 8 else i]):
                if kind in ("d2h", "both"):
                    h_out[i * part:(i + 1) * part].copy_(d_b[i * part:(i + 1) * part], non_blocking=True)
        torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / reps
    print(f"{kind} x{k}: {dt*1e6:.0f} us per 16 MiB ({n/dt/1e9:.1f} GB/s per direction)", flush=True)
for rep in range(2):
    for kind in ("h2d", "d2h", "both"):
        for k in (1, 2, 4):
            run(kind, k)
