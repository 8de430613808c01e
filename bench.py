#!/usr/bin/env python
"""Benchmark of the B200 morphology hot path (driver contract in the task statement).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload cfg2]

Default workload = BASELINE.json configs[1] ("cfg2"), the config the metric is quoted on:
erosion AND dilation of one 4096x4096 u8 image (top half uniform random, bottom half a binary
mask of 400 seeded rectangles) for every window of the sweep {3,7,15,31,63,101}^2, 31x1, 1x31.
One step = those 16 operations. value = output Gpixel/s of the whole job (all ranks).

Inputs are resident in HBM before the timed region; every operation of a step reads a different
input copy and writes a different output buffer out of 32 rotating pairs (1 GiB total, > 8x the
126 MB L2), so no operation is served from L2 by its predecessor. A step is one CUDA graph; its 16
operations are independent, so the graph forks them over --streams (default 2) streams and one
kernel's ramp-up / tail overlaps its neighbours. Per-window numbers ("per_window") are measured
separately, one operation at a time. Device time is measured with CUDA events on the launching
stream; multi-GPU time is the max over ranks.

Other workloads (for profiling / the scaling run): cfg1, cfg3 (transposes), cfg4 (512 x 1024^2
u16 opening 21x21, batch sharded over ranks), cfg5 (32768^2 u8 dilation 63x63, row bands +
halo exchange over NCCL).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2002_09474_b200.synth import CFG2_WINDOWS, cfg2_image, generate  # noqa: E402

METRIC = "erosion/dilation Gpixel/s (uint8, per window size) and achieved HBM GB/s vs peak"
ERODE, DILATE, OPEN, CLOSE, GRADIENT = 0, 1, 2, 3, 4
FALLBACK_HBM_GBS = 6650.0


# ---------------------------------------------------------------------------------------------
def parse_args(argv=None):
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--workload", default="cfg2", choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--e2e-threads", type=int, default=2,
                   help="host threads issuing the step's independent plugin calls in the e2e leg (each call stays "
                        "synchronous; two callers keep both PCIe directions busy)")
    p.add_argument("--eager", action="store_true", help="launch each op from Python instead of a CUDA graph")
    p.add_argument("--steps-per-graph", type=int, default=0,
                   help="steps captured into one CUDA graph (0 = as many as the rotating buffers allow and "
                        "--steps divides into; each stream walks its share of every step, joined once per graph)")
    p.add_argument("--streams", type=int, default=2,
                   help="streams the step graph forks its independent operations over (1 = serial)")
    p.add_argument("--soak-seconds", type=float, default=1.5)
    p.add_argument("--no-self-check", action="store_true",
                   help="skip the bit-exact check of the timed outputs against the CPU reference")
    p.add_argument("--dry-run", action="store_true",
                   help="CPU only (gloo): exercise the N-rank launch, barriers and max-over-ranks timing "
                        "with the oracle as the step; no GPU, no kernel")
    return p.parse_args(argv)


def maybe_spawn(args, argv) -> int | None:
    """`bench.py --gpus N` outside torchrun starts N ranks itself (torch.distributed.run, one
    process per GPU, rendezvous on 127.0.0.1) and returns their exit code; None = already a rank."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + list(argv)
    return subprocess.call(cmd)


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md, MEASURED_PEAKS.json absent)"


class Dist:
    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None
        self.backend = None

    def init(self, backend="nccl"):
        self.backend = backend
        if self.world > 1:
            import torch.distributed as dist
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            dist.init_process_group(backend=backend)
            self.pg = dist

    def barrier(self):
        if self.pg is not None:
            self.pg.barrier()

    def max(self, x: float) -> float:
        if self.pg is None:
            return x
        import torch
        on_gpu = self.backend == "nccl" and torch.cuda.is_available()
        t = torch.tensor([x], dtype=torch.float64, device="cuda" if on_gpu else "cpu")
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.pg is not None:
            self.pg.destroy_process_group()


# ---------------------------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled while the GPU is loaded (B200_PROFILING.md)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,utilization.gpu,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.file = None

    def start(self):
        try:
            self.file = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.dev}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=self.file, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.file.flush()
        rows = []
        with open(self.file.name) as f:
            for line in f:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) < 10:
                    continue
                try:
                    rows.append(dict(sm=float(parts[1]), smax=float(parts[2]), util=float(parts[4]),
                                     hw=parts[6], hwt=parts[7], swt=parts[8], pcap=parts[9]))
                except ValueError:
                    continue
        os.unlink(self.file.name)
        loaded = [r for r in rows if r["util"] >= 50] or rows
        reasons = set()
        for r in loaded:
            for key, name in (("hw", "hw_slowdown"), ("hwt", "hw_thermal_slowdown"), ("swt", "sw_thermal_slowdown"),
                              ("pcap", "sw_power_cap")):
                if r[key].lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median([r["sm"] for r in loaded]) if loaded else None,
                "sm_max_mhz": max(r["smax"] for r in loaded) if loaded else None,
                "reasons": sorted(reasons), "samples": len(loaded)}


# ---------------------------------------------------------------------------------------------
# Workloads. Each exposes: ops (list of (label, launch_fn, algorithmic_bytes, out_pixels)),
# e2e_step() -> (h2d, d2h) bytes, ref_step(nthreads) for the CPU legs, config dict.
# ---------------------------------------------------------------------------------------------
class Cfg2:
    name = "cfg2"
    dtype = "u8"
    NB = 32  # rotating input/output pairs (32 x 2 x 16 MiB = 1 GiB)

    def __init__(self, dist: Dist):
        self.dist = dist
        self.img = cfg2_image()
        self.size = self.img.shape[0]
        self.ops_list = [(wx, wy, op) for (wx, wy) in CFG2_WINDOWS for op in (ERODE, DILATE)]

    def setup_device(self):
        import torch
        import paper_2002_09474_b200 as pkg
        self.pkg = pkg
        base = torch.from_numpy(self.img).cuda()
        self.inputs = [base.clone() for _ in range(self.NB)]
        self.outputs = [torch.empty_like(base) for _ in range(self.NB)]
        self.cursor = 0
        self.written = {}
        n = self.size * self.size
        self.ops = []
        for (wx, wy, op) in self.ops_list:
            self.ops.append((f"{'erode' if op == ERODE else 'dilate'} {wx}x{wy}", (wx, wy, op), 2 * n, n))

    def launch(self, spec):
        wx, wy, op = spec
        i = self.cursor % self.NB
        self.cursor += 1
        self.written[i] = spec
        self.pkg.morph_device(self.inputs[i], self.outputs[i], wx, wy, op)

    def self_check(self) -> dict:
        """Every output buffer of the timed step graphs against the reference (all host threads):
        bit-exact or the run is reported as failed."""
        import torch
        R, port, nthreads = _reference_checker(self)
        if R is None:
            import oracle
            R, nthreads = oracle.restatement(), 1
        want = {}
        bad = []
        torch.cuda.synchronize()
        for i, spec in sorted(self.written.items()):
            if spec not in want:
                wx, wy, op = spec
                want[spec] = (R.morph(self.img, wx, wy, op, nthreads=nthreads) if nthreads > 1
                              else R.morph(self.img, wx, wy, op))
            if not np.array_equal(self.outputs[i].cpu().numpy(), want[spec]):
                bad.append({"buffer": i, "op": list(spec)})
        return {"checked_outputs": len(self.written), "distinct_ops": len(want), "bit_exact": not bad,
                "mismatches": bad[:8], "against": "reference (oracle/_ref)" if nthreads > 1 else "restatement"}

    def config(self):
        return {"workload": "cfg2: 4096x4096 u8, erode+dilate per window, windows "
                            + ",".join(f"{a}x{b}" for a, b in CFG2_WINDOWS),
                "image": "4096x4096 u8: rows 0-2047 seeded uniform (splitmix64 seed 2), rows 2048-4095 "
                         "0/255 mask of 400 seeded rectangles side 5-200",
                "ops_per_step": len(self.ops_list), "border": "replicate",
                "l2": "no flush: 32 rotating input/output buffer pairs (1 GiB) >> 126 MB L2",
                "parallelism": f"replicas x{self.dist.world} (independent images, no collective)"}

    def e2e_setup(self, threads=1):
        import concurrent.futures as cf
        import torch
        self.h_in = torch.from_numpy(self.img).pin_memory()
        # one pinned output image per calling thread (the calls of a step are independent)
        self.e2e_threads = max(1, threads)
        self.h_outs = [torch.empty_like(self.h_in).pin_memory() for _ in range(self.e2e_threads)]
        self.h_out = self.h_outs[0]
        self.e2e_pool = cf.ThreadPoolExecutor(self.e2e_threads) if self.e2e_threads > 1 else None

    def e2e_step(self):
        import ctypes as C
        L = self.pkg.lib()
        h, w = self.img.shape

        def run(t):  # thread t issues ops t, t + T, ...: synchronous C-ABI calls (ctypes drops the GIL)
            out = self.h_outs[t]
            for (wx, wy, op) in self.ops_list[t::self.e2e_threads]:
                rc = L.rmgpu_morph_host_u8(C.c_void_p(self.h_in.data_ptr()), w, C.c_void_p(out.data_ptr()), w,
                                           w, h, wx, wy, op, 0, 0, 0, 0)
                if rc:
                    raise RuntimeError(f"rmgpu_morph_host_u8 failed: {rc} {L.rmgpu_last_error()}")

        if self.e2e_pool:
            for f in [self.e2e_pool.submit(run, t) for t in range(self.e2e_threads)]:
                f.result()
        else:
            run(0)
        nb = len(self.ops_list) * h * w
        return nb, nb

    def out_pixels_per_step(self):
        return len(self.ops_list) * self.size * self.size

    # CPU legs (reference code, oracle/_ref): one full step = the same 16 operations
    def ref_step(self, R, nthreads, out, th=69, tv=59):
        for (wx, wy, op) in self.ops_list:
            R.morph(self.img, wx, wy, op, threshold_h=th, threshold_v=tv, nthreads=nthreads, out=out)
        return self.out_pixels_per_step()


class Cfg1(Cfg2):
    name = "cfg1"

    def __init__(self, dist: Dist):
        self.dist = dist
        self.img = generate(1920, 1080, 1)
        self.ops_list = [(3, 3, ERODE), (3, 3, DILATE)]

    def setup_device(self):
        import torch
        import paper_2002_09474_b200 as pkg
        self.pkg = pkg
        base = torch.from_numpy(self.img).cuda()
        self.NB = 64
        self.inputs = [base.clone() for _ in range(self.NB)]
        self.outputs = [torch.empty_like(base) for _ in range(self.NB)]
        self.cursor = 0
        self.written = {}
        n = self.img.size
        self.ops = [(f"{'erode' if op == ERODE else 'dilate'} 3x3", (wx, wy, op), 2 * n, n)
                    for (wx, wy, op) in self.ops_list]

    def config(self):
        return {"workload": "cfg1: 1920x1080 u8 erode+dilate 3x3 (seed 1)", "border": "replicate",
                "l2": "no flush: 64 rotating buffer pairs (265 MB) > L2",
                "parallelism": f"replicas x{self.dist.world}"}

    def out_pixels_per_step(self):
        return 2 * self.img.size


class Cfg4:
    """512 u16 1024x1024 images (seed 4, stream = image index), opening 21x21 replicate, batch sharded
    over the ranks (contiguous shards, no collective). One step = the rank's whole shard."""
    e2e_path = ("pinned host shard -> device in chunks of 64 images (H2D), morph_batched_device opening per chunk, "
                "D2H; three streams, synchronised at the end of the step")
    name = "cfg4"
    dtype = "u16"
    graphable = False
    N_IMAGES, SIZE, WIN = 512, 1024, 21

    def __init__(self, dist: Dist):
        from paper_2002_09474_b200.shard import batch_shard
        self.dist = dist
        self.first, self.count = batch_shard(self.N_IMAGES, dist.world, dist.rank)
        self.img = generate(self.SIZE, self.SIZE, 4, self.first, np.uint16)  # CPU-leg sample image

    def setup_device(self):
        import torch
        import paper_2002_09474_b200 as pkg
        self.pkg = pkg
        n = self.SIZE
        self.src = torch.empty((self.count, n, n), dtype=torch.uint16, device="cuda")
        self.dst = torch.empty_like(self.src)
        for k in range(self.count):
            pkg.generate_device(self.src[k], 4, self.first + k)
        npx = self.count * n * n
        self.ops = [(f"opening {self.WIN}x{self.WIN} x{self.count}", None, 4 * npx, npx)]

    def launch(self, spec):
        self.pkg.morph_batched_device(self.src, self.dst, self.WIN, self.WIN, OPEN)

    def config(self):
        return {"workload": f"cfg4: {self.N_IMAGES} x 1024x1024 u16 opening {self.WIN}x{self.WIN} (seed 4, "
                            "stream = image index), batch sharded", "images_this_rank": self.count,
                "border": "replicate", "l2": f"no flush: {self.count} x 2 MiB inputs >> L2 (G small)",
                "parallelism": f"batch shards x{self.dist.world} (no collective)"}

    def out_pixels_per_step(self):
        return self.count * self.SIZE * self.SIZE

    def e2e_setup(self):
        import torch
        self.h_in = self.src.cpu().pin_memory()
        self.h_out = torch.empty_like(self.h_in).pin_memory()

    def e2e_step(self):
        # the shard in chunks of 64 images over three streams: the upload of chunk k+1, the opening of
        # chunk k and the download of chunk k-1 overlap (both PCIe directions busy)
        import torch
        if not hasattr(self, "e2e_streams"):
            self.e2e_streams = [torch.cuda.Stream() for _ in range(3)]
            self.e2e_din = torch.empty_like(self.src)
            self.e2e_dout = torch.empty_like(self.src)
        up, run, down = self.e2e_streams
        main = torch.cuda.current_stream()
        for st in (up, run, down):
            st.wait_stream(main)
        step = 64
        for k0 in range(0, self.count, step):
            k1 = min(self.count, k0 + step)
            with torch.cuda.stream(up):
                self.e2e_din[k0:k1].copy_(self.h_in[k0:k1], non_blocking=True)
                ev_up = torch.cuda.Event()
                ev_up.record(up)
            with torch.cuda.stream(run):
                run.wait_event(ev_up)
                self.pkg.morph_batched_device(self.e2e_din[k0:k1], self.e2e_dout[k0:k1], self.WIN, self.WIN, OPEN,
                                              stream=run)
                ev_run = torch.cuda.Event()
                ev_run.record(run)
            with torch.cuda.stream(down):
                down.wait_event(ev_run)
                self.h_out[k0:k1].copy_(self.e2e_dout[k0:k1], non_blocking=True)
        torch.cuda.synchronize()
        nbytes = self.h_in.numel() * 2
        return nbytes, nbytes

    def self_check(self) -> dict:
        """Three images of the timed batch (first, middle, last) against the restatement."""
        import oracle
        from oracle import VANHERK
        R = oracle.restatement()
        bad = []
        picks = sorted({0, self.count // 2, self.count - 1}) if self.count else []
        for k in picks:
            src = R.generate(self.SIZE, self.SIZE, 4, self.first + k, np.uint16)
            got = self.dst[k].contiguous().view(torch_u8()).cpu().numpy().view(np.uint16)
            if not np.array_equal(got, R.morph(src, self.WIN, self.WIN, OPEN, h_algo=VANHERK, v_algo=VANHERK)):
                bad.append(self.first + k)
        return {"checked_images": [self.first + k for k in picks], "bit_exact": not bad, "mismatches": bad,
                "against": "restatement (u16: no reference)"}

    ref_port = True  # u16: the reference is u8-only; the CPU leg is the oracle restatement

    def ref_step(self, R, nthreads, out, th=69, tv=59):
        R.morph(self.img, self.WIN, self.WIN, OPEN)
        return self.SIZE * self.SIZE


class Cfg5:
    """32768^2 u8 (seed 5) dilation 63x63 replicate, split into G row bands; each step exchanges the
    31-row halos with the neighbouring ranks (NCCL point-to-point) and computes the band."""
    e2e_path = ("one rank: C-ABI rmgpu_morph_host_u8 on the whole pinned image (synchronous, pipelined over row "
                "bands); several ranks: pinned host band+halo -> device (H2D), halo exchange + morph_band, D2H")
    name = "cfg5"
    dtype = "u8"
    graphable = False
    SIZE, WIN = 32768, 63

    def __init__(self, dist: Dist):
        from paper_2002_09474_b200.shard import band_plan
        self.dist = dist
        self.band = band_plan(self.SIZE, dist.world, dist.rank, self.WIN // 2)
        self.img = generate(4096, 4096, 5)  # CPU-leg sample (a 4096^2 crop-sized image)

    def setup_device(self):
        import torch
        import paper_2002_09474_b200 as pkg
        self.pkg = pkg
        b = self.band
        full = torch.empty((self.SIZE, self.SIZE), dtype=torch.uint8, device="cuda")
        pkg.generate_device(full, 5)
        self.buf = full[b.in_y0:b.in_y0 + b.buffer_rows].clone()
        del full
        torch.cuda.empty_cache()
        self.out = torch.empty((b.rows, self.SIZE), dtype=torch.uint8, device="cuda")
        npx = b.rows * self.SIZE
        self.ops = [(f"dilate {self.WIN}x{self.WIN} band {b.rows} rows (+{b.above}/{b.below} halo)", None, 2 * npx,
                     npx)]

    def launch(self, spec):
        from paper_2002_09474_b200.shard import morph_band, morph_band_overlapped
        if self.dist.world > 1:  # interior rows computed while the halos fly, edge rows after
            morph_band_overlapped(self.buf, self.out, self.band, self.dist.world, self.dist.rank, self.WIN,
                                  self.WIN, DILATE, dist=self.dist.pg)
        else:
            morph_band(self.buf, self.out, self.band, self.WIN, self.WIN, DILATE)

    def self_check(self) -> dict:
        """Two 512-row crops of the band (first and last rows) against the reference on the same
        input rows plus their halo (exact: a band's rows see only the rows they would see whole)."""
        R, port, nthreads = _reference_checker(self)
        if R is None:
            return {"bit_exact": None, "note": "reference not built"}
        b, g = self.band, self.WIN // 2
        bad, crops = [], []
        for r0 in sorted({0, max(0, b.rows - 512)}):
            r1 = min(b.rows, r0 + 512)
            a = max(0, b.above + r0 - g)
            z = min(b.buffer_rows, b.above + r1 + g)
            host = self.buf[a:z].cpu().numpy()
            want = R.morph(host, self.WIN, self.WIN, DILATE, nthreads=nthreads)[b.above + r0 - a:b.above + r1 - a]
            crops.append([b.y0 + r0, b.y0 + r1])
            if not np.array_equal(self.out[r0:r1].cpu().numpy(), want):
                bad.append([b.y0 + r0, b.y0 + r1])
        return {"checked_rows": crops, "bit_exact": not bad, "mismatches": bad, "against": "reference (oracle/_ref)"}

    def config(self):
        return {"workload": f"cfg5: {self.SIZE}x{self.SIZE} u8 dilate {self.WIN}x{self.WIN} (seed 5), row bands",
                "band_rows_this_rank": self.band.rows, "halo_rows": [self.band.above, self.band.below],
                "border": "replicate", "l2": "no flush: 1 GiB image >> L2",
                "parallelism": f"row bands x{self.dist.world}, {self.WIN // 2}-row halo exchange per step "
                               "(NCCL send/recv)"}

    def out_pixels_per_step(self):
        return self.band.rows * self.SIZE

    def e2e_setup(self):
        import torch
        self.h_in = self.buf.cpu().pin_memory()
        self.h_out = torch.empty_like(self.out, device="cpu").pin_memory()

    def e2e_step(self):
        import torch
        if self.dist.world == 1:
            # one rank: the band is the whole image -- the synchronous C-ABI host call (it pipelines
            # the upload, the kernels and the download over row bands itself)
            import ctypes as C
            L = self.pkg.lib()
            n = self.SIZE
            rc = L.rmgpu_morph_host_u8(C.c_void_p(self.h_in.data_ptr()), n, C.c_void_p(self.h_out.data_ptr()), n,
                                       n, n, self.WIN, self.WIN, DILATE, 0, 0, 0, 0)
            if rc:
                raise RuntimeError(f"rmgpu_morph_host_u8 failed: {rc} {L.rmgpu_last_error()}")
            return self.h_in.numel(), self.h_out.numel()
        self.buf.copy_(self.h_in, non_blocking=True)
        self.launch(None)
        self.h_out.copy_(self.out, non_blocking=True)
        torch.cuda.synchronize()
        return self.h_in.numel(), self.h_out.numel()

    def ref_step(self, R, nthreads, out, th=69, tv=59):
        R.morph(self.img, self.WIN, self.WIN, DILATE, threshold_h=th, threshold_v=tv, nthreads=nthreads, out=out)
        return self.img.size


class Cfg3:
    """Standalone transposes: 8192^2 u8 and u16 images, 2^24 8x8 and 2^24 16x16 u8 tiles in place."""
    e2e_path = "pinned 8192^2 u8 -> device (H2D), transpose_device, D2H, synchronised"
    name = "cfg3"
    dtype = "u8/u16"
    graphable = True
    NB = 4

    def __init__(self, dist: Dist):
        self.dist = dist
        self.img = generate(2048, 2048, 3)

    def setup_device(self):
        import torch
        import paper_2002_09474_b200 as pkg
        self.pkg = pkg
        n = 8192
        # 4 rotating u8 pairs (512 MiB) and 2 u16 pairs (512 MiB): no image transpose re-reads its
        # input or output from the 126 MB L2
        self.a8s = [torch.empty((n, n), dtype=torch.uint8, device="cuda") for _ in range(4)]
        self.a16s = [torch.empty((n, n), dtype=torch.uint16, device="cuda") for _ in range(2)]
        for a in self.a8s:
            pkg.generate_device(a, 3)
        for a in self.a16s:
            pkg.generate_device(a, 30)
        self.t8s = [torch.empty_like(a) for a in self.a8s]
        self.t16s = [torch.empty_like(a) for a in self.a16s]
        self.a8, self.a16, self.t8, self.t16 = self.a8s[0], self.a16s[0], self.t8s[0], self.t16s[0]
        self.k8 = self.k16 = 0
        self.tiles8 = torch.empty((1 << 24) * 64, dtype=torch.uint8, device="cuda")
        self.tiles16 = torch.empty((1 << 24) * 256, dtype=torch.uint8, device="cuda")
        pkg.generate_device(self.tiles8.view(1 << 14, -1), 31)
        pkg.generate_device(self.tiles16.view(1 << 16, -1), 32)
        self.cursor = 0
        e = n * n
        self.ops = [("transpose 8192^2 u8", "t8", 2 * e, e), ("transpose 8192^2 u16", "t16", 4 * e, e),
                    ("2^24 tiles 8x8 u8 in place", "k8", 2 * (1 << 24) * 64, (1 << 24) * 64),
                    ("2^24 tiles 16x16 u8 in place", "k16", 2 * (1 << 24) * 256, (1 << 24) * 256)]

    def launch(self, spec):
        if spec == "t8":
            i = self.k8 % len(self.a8s)
            self.k8 += 1
            self.pkg.transpose_device(self.a8s[i], self.t8s[i])
        elif spec == "t16":
            i = self.k16 % len(self.a16s)
            self.k16 += 1
            self.pkg.transpose_device(self.a16s[i], self.t16s[i])
        elif spec == "k8":
            self.pkg.transpose_tiles_device(self.tiles8, 8)
        else:
            self.pkg.transpose_tiles_device(self.tiles16, 16)

    def self_check(self) -> dict:
        """Image transposes: every element against x^T. Tiles: transposed an even number of times
        by the timed steps (in place), so they must equal their generator input again; plus one
        extra call checked per element against the closed form."""
        import torch
        torch.cuda.synchronize()
        ok = all(bool(torch.equal(t, a.t().contiguous())) for a, t in zip(self.a8s, self.t8s))
        ok &= all(bool(torch.equal(t.view(torch.uint8).view(8192, 8192, 2),
                                   a.view(torch.uint8).view(8192, 8192, 2).transpose(0, 1).contiguous()))
                  for a, t in zip(self.a16s, self.t16s))
        for t, n in ((self.tiles8, 8), (self.tiles16, 16)):
            before = t.view(-1, n, n)[:1 << 16].transpose(1, 2).contiguous()
            self.pkg.transpose_tiles_device(t, n)
            torch.cuda.synchronize()
            ok &= bool(torch.equal(t.view(-1, n, n)[:1 << 16], before))
            self.pkg.transpose_tiles_device(t, n)  # back
        return {"bit_exact": ok, "checked": "every rotating 8192^2 image pair (all elements); 2^16 tiles of each size",
                "against": "closed form (x^T)"}

    def config(self):
        return {"workload": "cfg3: transpose 8192^2 u8 + 8192^2 u16, 2^24 8x8 + 2^24 16x16 u8 tiles in place",
                "unit_note": "value counts transposed elements (Gelem/s)",
                "l2": "no flush: 4 rotating u8 and 2 u16 image pairs (512 MiB each), 1 / 4 GiB tile arrays >> L2",
                "parallelism": f"replicas x{self.dist.world}"}

    def out_pixels_per_step(self):
        return sum(o[3] for o in self.ops)

    def e2e_setup(self):
        import torch
        self.h_in = self.a8.cpu().pin_memory()
        self.h_out = torch.empty_like(self.h_in).pin_memory()

    def e2e_step(self):
        import torch
        d = self.h_in.to("cuda", non_blocking=True)
        o = torch.empty_like(d)
        self.pkg.transpose_device(d, o)
        self.h_out.copy_(o, non_blocking=True)
        torch.cuda.synchronize()
        return self.h_in.numel(), self.h_out.numel()

    def e2e_pixels_per_step(self):
        return self.a8.numel()  # the e2e leg moves and transposes the 8192^2 u8 image

    def ref_step(self, R, nthreads, out, th=69, tv=59):
        R.transpose_image(self.img, nthreads=nthreads)
        return self.img.size


def torch_u8():
    import torch
    return torch.uint8


WORKLOADS = {"cfg1": Cfg1, "cfg2": Cfg2, "cfg3": Cfg3, "cfg4": Cfg4, "cfg5": Cfg5}


# ---------------------------------------------------------------------------------------------
def _reference_checker(wl):
    """(checker, is_port, threads): the reference's own code (oracle/_ref) on every host thread,
    pinned one per CPU; for u16 (no reference) the restatement on one thread."""
    import oracle
    port = getattr(wl, "ref_port", False)
    if not port and not oracle.Reference.available():
        return None, port, 0
    if port:
        return oracle.restatement(), True, 1
    R = oracle.reference()
    R.set_pinning(True)
    return R, False, (os.cpu_count() or 1)


def _median_step(wl, R, nthreads, out, reps, **kw) -> tuple[float, int]:
    """timing::median_ns (timing.hpp:22-53): one warm-up, the median of `reps` timed steps."""
    wl.ref_step(R, nthreads, out, **kw)
    times, px = [], 0
    for _ in range(reps):
        t0 = time.perf_counter()
        px = wl.ref_step(R, nthreads, out, **kw)
        times.append(time.perf_counter() - t0)
    return statistics.median(times), px


def _cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference_arm(args, dist: Dist):
    """--impl reference: the reference's own CPU implementation (oracle/_ref, compiled from the
    reference sources) on the host cores, same workload/metric. Rank 0 only."""
    if dist.rank != 0:
        return 0
    wl = WORKLOADS[args.workload](dist)
    R, port, nthreads = _reference_checker(wl)
    if R is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/librmref.so not built"}))
        return 0
    out = np.empty_like(wl.img)
    for _ in range(max(0, args.warmup - 1)):
        wl.ref_step(R, nthreads, out)
    med, px = _median_step(wl, R, nthreads, out, max(1, args.steps))
    value = px / med / 1e9
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "Gpixel/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": med * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": wl.dtype,
            "data": "synthetic (seeded generator, SURVEY.md 8d)", "config": wl.config(),
            "cpu_baseline": {"value": value, "unit": "Gpixel/s", "cores": nthreads,
                             "kind": "port" if port else "reference", "cpu_model": _cpu_model(),
                             "timing": "median of the timed steps after one warm-up (timing.hpp:22-53)",
                             "sample": (f"one {wl.name} image per step through the oracle restatement (u16 has no "
                                        "reference implementation), 1 thread") if port else
                                       (f"{wl.name} sample per step; reference rectmorph (oracle/_ref, -O3, "
                                        f"DispatchConfig paper 69/59) on {nthreads} pinned threads via row bands")},
            "e2e": {"value": value, "unit": "Gpixel/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def cpu_baseline(wl) -> dict | None:
    """The reference on the host cores beside our numbers (reported, not a target): all threads
    (median of 5 steps), one thread (median of 3), and all threads with the thresholds the
    reference's own calibrate() picks on this host (dispatch.cpp:180-248)."""
    try:
        R, port, nthreads = _reference_checker(wl)
    except Exception:
        return None
    if R is None:
        return None
    out = np.empty_like(wl.img)
    med, px = _median_step(wl, R, nthreads, out, 5)
    res = {"value": px / med / 1e9, "unit": "Gpixel/s", "cores": nthreads, "kind": "port" if port else "reference",
           "cpu_model": _cpu_model(), "timing": "median of 5 steps after one warm-up (timing.hpp:22-53)",
           "sample": f"{wl.name} CPU sample ({px} output px per step) through "
                     + ("the oracle restatement (u16: no reference), 1 thread" if port else
                        f"the reference rectmorph (oracle/_ref, DispatchConfig paper 69/59) on {nthreads} pinned "
                        "host threads (row bands + halo)")}
    if not port:
        med1, _ = _median_step(wl, R, 1, out, 3)
        res["single_thread"] = {"ms_per_step": med1 * 1e3, "value": px / med1 / 1e9}
        if wl.name != "cfg3":
            th, tv = R.calibrate(1024, 1024, list(range(3, 128, 8)), 3)
            medc, _ = _median_step(wl, R, nthreads, out, 5, th=th, tv=tv)
            res["calibrated"] = {"threshold_h": th, "threshold_v": tv, "value": px / medc / 1e9,
                                 "ms_per_step": medc * 1e3,
                                 "how": "reference calibrate(1024, 1024, windows 3..127 step 8, reps 3) on this host"}
    return res


def run_dry(args, dist: Dist) -> int:
    """--dry-run: the multi-rank plumbing on CPU (gloo): every rank runs a small oracle morphology as
    its step between barriers, the time is the max over ranks, rank 0 prints the contract line."""
    import oracle
    dist.init("gloo")
    R = oracle.restatement()
    img = R.generate(512, 512, 100 + dist.rank)
    for _ in range(args.warmup):
        R.morph(img, 15, 15, ERODE)
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        R.morph(img, 15, 15, ERODE)
    dist.barrier()
    dt = dist.max(time.perf_counter() - t0)
    if dist.rank == 0:
        print(json.dumps({"metric": METRIC, "value": dist.world * img.size * args.steps / dt / 1e9,
                          "unit": "Gpixel/s", "n_gpus": dist.world, "steps": args.steps, "warmup": args.warmup,
                          "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
                          "vs_baseline": None, "dtype": "u8", "data": "synthetic", "dry_run": True,
                          "config": {"workload": "dry run: 512x512 u8 erode 15x15 per rank through the CPU oracle"}}))
    dist.close()
    return 0


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    args = parse_args(argv)
    rc = maybe_spawn(args, argv)
    if rc is not None:
        return rc
    dist = Dist()
    if args.dry_run:
        return run_dry(args, dist)
    if args.impl == "reference":
        return run_reference_arm(args, dist)

    import torch
    import paper_2002_09474_b200 as pkg
    torch.cuda.set_device(dist.local)
    dist.init("nccl")
    wl = WORKLOADS[args.workload](dist)
    wl.setup_device()
    stream = torch.cuda.current_stream()
    peak, peak_src = peaks()

    nops = len(wl.ops)
    slots = max(1, getattr(wl, "NB", nops) // nops)  # steps the rotating buffers hold
    spg = 1
    if not args.eager and getattr(wl, "graphable", True):
        want = args.steps_per_graph if args.steps_per_graph > 0 else min(slots, 32)
        spg = max(d for d in range(1, max(1, min(want, slots, args.steps)) + 1) if args.steps % d == 0)
    ngraphs = max(1, slots // spg)
    use_graphs = not args.eager and getattr(wl, "graphable", True)

    def eager_step():
        for (_, spec, _, _) in wl.ops:
            wl.launch(spec)

    for _ in range(max(args.warmup, 0)):  # warm-up also fills the launch caches before capture
        eager_step()
    torch.cuda.synchronize()

    # One CUDA graph per step (16 kernel nodes; one graph per rotating-buffer assignment), so the
    # timed region measures the kernels, not Python/ctypes launch latency.
    graphs, glaunch = [], 0
    if use_graphs:
        cap = torch.cuda.Stream()
        wl.cursor = 0
        for _ in range(ngraphs):
            g = torch.cuda.CUDAGraph()
            l0 = pkg.launch_count()
            with torch.cuda.graph(g, stream=cap):
                if args.streams > 1:
                    # the operations of a step are independent: fork them over several streams so
                    # one kernel's ramp-up / tail overlaps its neighbours (joined at the end)
                    side = [torch.cuda.Stream() for _ in range(args.streams - 1)]
                    fork = torch.cuda.Event()
                    fork.record(cap)
                    for sd in side:
                        sd.wait_event(fork)
                    lanes = [cap] + side
                    nl = len(lanes)
                    # lane i takes ops i, i+nl, ...; odd lanes walk their share in reverse so that
                    # concurrently running kernels differ (small-window K1 beside large-window K2)
                    for i, lane_s in enumerate(lanes):
                        share = list(range(i, len(wl.ops), nl))
                        if i % 2:
                            share.reverse()
                        with torch.cuda.stream(lane_s):
                            for _ in range(spg):  # the graph's steps are independent batches too
                                for k in share:
                                    wl.launch(wl.ops[k][1])
                    for sd in side:
                        ev = torch.cuda.Event()
                        ev.record(sd)
                        cap.wait_event(ev)
                else:
                    for _ in range(spg):
                        eager_step()
            glaunch = pkg.launch_count() - l0
            graphs.append(g)
        for g in graphs:
            g.replay()
        torch.cuda.synchronize()

    def step(i):  # spg steps per call when graphs are on
        if graphs:
            graphs[i % len(graphs)].replay()
        else:
            eager_step()

    sampler = ClockSampler(torch.cuda.current_device())
    sampler.start()
    t_soak = time.perf_counter()
    while time.perf_counter() - t_soak < args.soak_seconds:  # keep the GPU loaded for the sampler
        for i in range(20):
            step(i)
        torch.cuda.synchronize()

    evs = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    dist.barrier()
    torch.cuda.synchronize()
    launches0 = pkg.launch_count()
    evs[0].record(stream)
    for i in range(args.steps // spg):
        step(i)
    evs[1].record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    launches = pkg.launch_count() - launches0 + (glaunch * (args.steps // spg) if graphs else 0)
    clocks = sampler.stop()

    total_ms = evs[0].elapsed_time(evs[1])
    max_ms = dist.max(total_ms)
    ms_per_step = max_ms / args.steps
    value = dist.world * wl.out_pixels_per_step() * args.steps / (max_ms / 1e3) / 1e9

    # the timed steps' outputs, bit-exact against the CPU reference (outside the timed region,
    # before the per-operation timings below overwrite the buffers)
    check = None
    if dist.rank == 0 and not args.no_self_check and hasattr(wl, "self_check"):
        check = wl.self_check()

    def family(label, spec) -> str:
        if wl.name in ("cfg1", "cfg2"):
            return pkg.plan_name(1, wl.img.shape[1], wl.img.shape[0], spec[0], spec[1], spec[2]).split("_")[0]
        return label.split(" ")[0] if wl.name != "cfg3" else ("tiles" if "tiles" in label else "image")

    # per-operation durations: a graph of NB launches of one operation over all rotating buffers
    per_window = []
    tot_b = tot_t = 0.0
    fam_b, fam_t, fam_ops = {}, {}, {}
    for (label, spec, nbytes, npx) in wl.ops:
        nb = getattr(wl, "NB", 1) if graphs else 3
        wl.cursor = 0
        if graphs:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=cap):
                for _ in range(nb):
                    wl.launch(spec)
            g.replay()
            torch.cuda.synchronize()
            reps = max(1, 64 // nb)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(reps):
                g.replay()
            e1.record(stream)
            torch.cuda.synchronize()
            n = reps * nb
        else:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            n = nb
            e0.record(stream)
            for _ in range(n):
                wl.launch(spec)
            e1.record(stream)
            torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / n
        tot_b += nbytes
        tot_t += ms
        fam = family(label, spec)
        fam_b[fam] = fam_b.get(fam, 0) + nbytes
        fam_t[fam] = fam_t.get(fam, 0) + ms
        fam_ops.setdefault(fam, []).append(label)
        per_window.append({"op": label, "kernel": fam, "us": round(ms * 1e3, 2),
                           "gpix_s": round(npx / (ms / 1e3) / 1e9, 1), "gb_s": round(nbytes / (ms / 1e3) / 1e9, 1),
                           "frac": round(nbytes / (ms / 1e3) / 1e9 / peak, 3)})
    # roofline of the dominant kernel: the family with the largest share of the per-operation
    # device time; achieved = its algorithmic bytes / its device time (CUDA events, serial)
    dom = max(fam_t, key=fam_t.get)
    achieved = fam_b[dom] / (fam_t[dom] / 1e3) / 1e9
    step_bytes = sum(o[2] for o in wl.ops)
    step_gbs = dist.world * step_bytes / (ms_per_step / 1e3) / 1e9

    traffic, traffic_src = None, None
    tpath = os.path.join(ROOT, "profiles", f"traffic_{wl.name}.json")
    if os.path.exists(tpath):
        try:
            tj = json.load(open(tpath))
            per_op = tj.get("per_op") or {}
            vals = [per_op[lab]["dram_bytes"] for lab in fam_ops[dom] if lab in per_op]
            if vals:
                traffic = sum(vals) / len(vals)
                traffic_src = f"{tpath[len(ROOT) + 1:]}: ncu dram__bytes_read+write per op, mean over {len(vals)} ops"
            elif tj.get("bytes_per_launch"):
                traffic = tj["bytes_per_launch"]
                traffic_src = tpath[len(ROOT) + 1:]
        except Exception:
            traffic = None

    e2e = None
    if not args.no_e2e:
        import inspect
        if "threads" in inspect.signature(wl.e2e_setup).parameters:
            wl.e2e_setup(threads=args.e2e_threads)
        else:
            wl.e2e_setup()
        wl.e2e_step()  # warm host pool / pinned paths
        wl.e2e_step()
        dist.barrier()
        t0 = time.perf_counter()
        h2d = d2h = 0
        for _ in range(args.steps):
            a, b = wl.e2e_step()
            h2d, d2h = a, b
        e2e_s = dist.max(time.perf_counter() - t0)
        e2e_px = getattr(wl, "e2e_pixels_per_step", wl.out_pixels_per_step)()
        e2e = {"value": dist.world * e2e_px * args.steps / e2e_s / 1e9, "unit": "Gpixel/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "path": getattr(wl, "e2e_path", "C-ABI rmgpu_morph_host_u8 per op (pinned host buffers; the call "
                                                 "pipelines H2D, kernels and D2H over row bands; synchronous; the "
                                                 f"step's independent calls issued from {getattr(wl, 'e2e_threads', 1)} "
                                                 "host thread(s))")}

    cpu = None
    if dist.rank == 0 and dist.world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(wl)

    if dist.rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "Gpixel/s", "n_gpus": dist.world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": wl.dtype,
                "data": "synthetic (seeded counter-based generator, SURVEY.md 8d; no dataset named)",
                "config": wl.config(),
                "launch": (f"CUDA graphs of {spg} step(s) ({glaunch} kernel nodes per graph, the independent "
                           f"operations forked over {args.streams} streams, joined once per graph)") if graphs else "eager",
                "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                             "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                             "kernel": f"{dom}: " + ", ".join(fam_ops[dom]),
                             "kernel_share_of_op_time": round(fam_t[dom] / tot_t, 3),
                             "how": "algorithmic bytes of the dominant kernel family's operations / their device "
                                    "time, each operation timed alone (CUDA events over a graph of launches)",
                             "algorithmic_bytes": "1 read + 1 write per output pixel (per element for transposes)",
                             "peak_source": peak_src,
                             "step": {"achieved": step_gbs, "frac": step_gbs / peak,
                                      "how": "all operations of the timed step (algorithmic bytes x ranks) / "
                                             "ms_per_step"},
                             "families": {f: {"achieved": fam_b[f] / (fam_t[f] / 1e3) / 1e9,
                                              "frac": fam_b[f] / (fam_t[f] / 1e3) / 1e9 / peak,
                                              "ops": len(fam_ops[f])} for f in fam_t}},
                "self_check": check,
                "per_window": per_window,
                "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks, "gpu_launches": launches,
                "plans": {lab: pkg.plan_name(1, 4096, 4096, spec[0], spec[1], spec[2]) for lab, spec, _, _ in wl.ops}
                if wl.name == "cfg2" else None}
        print(json.dumps(line))
    dist.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
