"""PCIe probe: H2D alone, D2H alone, both concurrently (pinned buffers, separate streams)."""
import time
import torch
n = 16 << 20
h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def run(kind, reps=20):
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
    print(f"{kind}: {dt*1e3:.3f} ms per 16 MiB ({n/dt/1e9:.1f} GB/s per direction)")
for k in ("h2d", "d2h", "both", "h2d", "d2h", "both"):
    run(k)
