"""Time morph ops under planner-knob settings in one process (CUDA graphs over rotating buffers > L2).
python tools/sweep.py "W H wx wy op elem" [...] --knob name=v1,v2 [--knob ...]
Knobs are rmgpu_debug_set overrides (e.g. sep_pf=1,2,3 sep_rb=40,80). Prints one line per setting."""
import itertools
import os
import sys

sys.path.insert(0, os.environ.get("PKGROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2002_09474_b200 as pkg  # noqa: E402
from paper_2002_09474_b200._native import lib  # noqa: E402

cases, knobs = [], []
args = sys.argv[1:]
i = 0
while i < len(args):
    if args[i] == "--knob":
        k, v = args[i + 1].split("=")
        knobs.append((k, [int(x) for x in v.split(",")]))
        i += 2
    else:
        cases.append(tuple(int(x) for x in args[i].split()))
        i += 1
peak = 6521.1


def run(case):
    W, H, wx, wy, op, elem = case
    dt = torch.uint8 if elem == 1 else torch.uint16
    nbytes = W * H * elem
    NB = max(2, min(32, int(1024e6 // (2 * nbytes))))
    srcs = [torch.empty((H, W), dtype=dt, device="cuda") for _ in range(NB)]
    for s in srcs:
        pkg.generate_device(s, 2)
    dsts = [torch.empty_like(s) for s in srcs]
    for k in range(NB):
        pkg.morph_device(srcs[k], dsts[k], wx, wy, op)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    with torch.cuda.graph(g, stream=st):
        for k in range(NB):
            pkg.morph_device(srcs[k], dsts[k], wx, wy, op)
    g.replay()
    torch.cuda.synchronize()
    reps = max(2, 64 // NB)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    best = 1e30
    for _ in range(3):
        ev[0].record()
        for _ in range(reps):
            g.replay()
        ev[1].record()
        torch.cuda.synchronize()
        best = min(best, ev[0].elapsed_time(ev[1]) / (reps * NB) * 1e3)
    del g
    return best, 2 * nbytes / best / 1e3


names = [k for k, _ in knobs]
for combo in itertools.product(*[v for _, v in knobs]) if knobs else [()]:
    for k, v in zip(names, combo):
        lib().rmgpu_debug_set(k.encode(), v)
    for case in cases:
        us, gbs = run(case)
        W, H, wx, wy, op, elem = case
        print(f"{W}x{H} {wx}x{wy} op{op} u{8*elem} {' '.join(f'{k}={v}' for k, v in zip(names, combo))}: "
              f"{us:8.2f} us {gbs:6.0f} GB/s {gbs/peak*100:5.1f}%  {pkg.plan_name(elem, W, H, wx, wy, op)}", flush=True)
    for k in names:
        lib().rmgpu_debug_set(k.encode(), -1)
