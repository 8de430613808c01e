"""Multi-GPU sharding of the morphology path: one process per GPU.

* Batch sharding (cfg4): independent images, contiguous shards; no collective.
* Row bands (cfg5): one giant image split into G row bands. Each rank keeps its band plus up to
  ``wing`` halo rows above and below (wing = wy // 2). One exchange step per operation: every rank
  sends its first ``wing`` rows to the rank above and its last ``wing`` rows to the rank below
  (point-to-point, one batched group: NCCL over NVLink on GPUs, gloo on CPU in the tests). The band is
  then computed with ``rmgpu_morph_band_*``: real neighbour rows at interior band edges, the border rule
  (replicate clamp / constant) only at the global top and bottom — bit-identical to computing the whole
  image at once, because every output row of the band sees exactly the input rows it would see there.

The functions here are pure host logic (plans, buffer slicing, the exchange); the per-band compute is
``api.morph_band_device``. Reference semantics: image.cpp:58-66 (border), separable.cpp:130-157.
"""
from __future__ import annotations

from dataclasses import dataclass


def batch_shard(n_images: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous shard of a batch: (first image, count). Shards differ by at most one image."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(n_images, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


@dataclass(frozen=True)
class Band:
    """Rows [y0, y0 + rows) of an image of height H, with halo rows above / below held locally."""
    y0: int
    rows: int
    above: int  # halo rows above the band held in the local buffer (0 at the global top)
    below: int  # halo rows below (0 at the global bottom)
    height: int

    @property
    def buffer_rows(self) -> int:
        return self.above + self.rows + self.below

    @property
    def in_y0(self) -> int:
        """Global row of local buffer row 0."""
        return self.y0 - self.above


def band_plan(height: int, world: int, rank: int, wing: int) -> Band:
    """Band of ``rank``: ceil-split rows, halo = min(wing, rows available beyond the band)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    per = -(-height // world)
    y0 = min(rank * per, height)
    rows = max(0, min(per, height - y0))
    above = min(wing, y0)
    below = min(wing, height - (y0 + rows))
    return Band(y0, rows, above, below, height)


def neighbours(world: int, rank: int, height: int) -> tuple[int | None, int | None]:
    """Ranks owning the non-empty bands directly above / below this one (None at the edges)."""
    up = rank - 1 if rank > 0 else None
    down = rank + 1 if rank + 1 < world and band_plan(height, world, rank + 1, 0).rows > 0 else None
    return up, down


def _halo_ops(buf, band: Band, world: int, rank: int, wing: int, dist, group):
    """The point-to-point ops of one exchange: receives go straight into the halo rows of ``buf``
    (contiguous row slices of the band buffer), sends read the band's first / last rows in place."""
    per = -(-band.height // world)
    if per < wing:
        raise ValueError(f"bands of {per} rows are thinner than the halo ({wing}); use fewer ranks")
    up, down = neighbours(world, rank, band.height)
    ops = []
    a, r = band.above, band.rows
    if up is not None:
        n_send = band_plan(band.height, world, up, wing).below  # the rank above holds our first rows
        ops.append(dist.P2POp(dist.isend, buf[a:a + n_send], up, group))
        ops.append(dist.P2POp(dist.irecv, buf[:a], up, group))
    if down is not None:
        n_send = band_plan(band.height, world, down, wing).above  # the rank below holds our last rows
        ops.append(dist.P2POp(dist.isend, buf[a + r - n_send:a + r], down, group))
        ops.append(dist.P2POp(dist.irecv, buf[a + r:], down, group))
    return ops


def start_halo_exchange(buf, band: Band, world: int, rank: int, wing: int, dist=None, group=None):
    """Issue the exchange (one batched isend / irecv group) and return its requests without
    waiting: with NCCL the transfers run on NCCL's stream while the caller keeps computing."""
    if dist is None:
        import torch.distributed as dist
    if band.rows == 0 or wing == 0 or world == 1:
        return []
    ops = _halo_ops(buf, band, world, rank, wing, dist, group)
    return dist.batch_isend_irecv(ops) if ops else []


def exchange_halos(buf, band: Band, world: int, rank: int, wing: int, dist=None, group=None) -> None:
    """Fill the halo rows of ``buf`` ([buffer_rows, W] tensor, band rows at [above, above+rows))
    from the neighbouring ranks: one batched point-to-point group (isend/irecv pairs), received
    directly into the halo rows.

    The rank above needs our first ``its below`` rows; the rank below needs our last ``its above``
    rows. Every band must hold at least ``wing`` rows (checked), so one hop suffices.
    """
    for req in start_halo_exchange(buf, band, world, rank, wing, dist, group):
        req.wait()


def interior_rows(band: Band, wing: int) -> tuple[int, int]:
    """Output rows [lo, hi) of the band (band-relative) whose windows stay inside the band's own
    rows or reach only the true image border: computable before the halos arrive."""
    lo = min(band.rows, wing if band.above > 0 else 0)
    hi = band.rows - (wing if band.below > 0 else 0)
    return lo, max(lo, hi)


def _band_pieces(buf, out, band: Band, wing: int, launch, halos_pending: bool, stage: str) -> None:
    """The interior rows (stage "interior": before the halos) or the edge rows (stage "edges":
    after them) of one band. Context rows past a window's reach are dropped by the C-ABI, so the
    edge pieces simply pass everything above / below them."""
    a, r, rows = band.above, band.rows, band.buffer_rows
    if not halos_pending:
        if stage == "interior":
            launch(buf, a, band.below, out)
        return
    lo, hi = interior_rows(band, wing)
    if stage == "interior":
        if hi > lo:
            ca = lo if a > 0 else 0          # band rows [0, lo) above the piece (none at the image top)
            cb = r - hi if band.below > 0 else 0
            launch(buf[a + lo - ca:a + hi + cb], ca, cb, out[lo:hi])
        return
    if lo > 0:  # top edge rows, the halo above now present
        launch(buf, a, rows - a - lo, out[0:lo])
    if hi < r:  # bottom edge rows, the halo below now present
        launch(buf, a + hi, rows - a - r, out[hi:r])


def morph_band_overlapped(buf, out, band: Band, world: int, rank: int, wx: int, wy: int, op: int,
                          border: int = 0, value: int = 0, dist=None, group=None, stream=None) -> None:
    """One band with the halo exchange overlapped: issue the exchange, compute
    the interior rows [wing, rows - wing) from the band's own rows while the halos fly, then the
    edge rows once they have arrived. Erode / dilate / gradient (one wing of halo)."""
    from .api import morph_band_device
    wing = wy // 2
    if band.rows == 0:
        return

    def launch(src, above, below, dst):
        morph_band_device(src, above, below, dst, wx, wy, op, border, value, stream)

    reqs = start_halo_exchange(buf, band, world, rank, wing, dist, group)
    _band_pieces(buf, out, band, wing, launch, bool(reqs), "interior")
    for req in reqs:
        req.wait()  # NCCL: the current stream waits for the transfers, the host does not
    _band_pieces(buf, out, band, wing, launch, bool(reqs), "edges")


def morph_band(buf, out, band: Band, wx: int, wy: int, op: int, border: int = 0, value: int = 0,
               stream=None) -> None:
    """GPU compute of one band (``buf`` holds halo + band rows on the device, ``out`` the band rows)."""
    from .api import morph_band_device
    if band.rows == 0:
        return
    morph_band_device(buf, band.above, band.below, out, wx, wy, op, border, value, stream)


def morph_bands_local(src, out, n_bands: int, wx: int, wy: int, op: int, border: int = 0, value: int = 0,
                      devices=None) -> None:
    """The row-band split driven from ONE process: band k lives in its own buffer on
    ``devices[k % len(devices)]`` (default: the source's device) holding only its own rows; the
    halos move between the band buffers by device-to-device copies (peer copies over NVLink
    across GPUs) on each band's stream while the interior rows are computed, then the edge rows.
    The same pipeline as the NCCL ranks (morph_band_overlapped), testable on one GPU.
    ``src`` / ``out``: [H, W] tensors; ``out`` receives every band. Erode / dilate / gradient."""
    import torch
    from .api import morph_band_device
    H = src.shape[0]
    wing = wy // 2
    devices = devices or [src.device]
    bands = [band_plan(H, n_bands, k, wing) for k in range(n_bands)]
    if any(0 < b.rows < wing for b in bands):
        raise ValueError("bands thinner than the halo: use fewer bands")
    bufs, outs, streams = [], [], []
    for k, b in enumerate(bands):
        dev = torch.device(devices[k % len(devices)])
        buf = torch.empty((b.buffer_rows,) + tuple(src.shape[1:]), dtype=src.dtype, device=dev)
        buf[b.above:b.above + b.rows].copy_(src[b.y0:b.y0 + b.rows])
        bufs.append(buf)
        outs.append(torch.empty((b.rows,) + tuple(src.shape[1:]), dtype=src.dtype, device=dev))
        streams.append(torch.cuda.Stream(device=dev))
    ready = []
    for k in range(n_bands):  # band rows in place before any stream reads a neighbour's
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(bufs[k].device))
        ready.append(ev)

    def launcher(k):
        def launch(s_, above, below, dst):
            morph_band_device(s_, above, below, dst, wx, wy, op, border, value, streams[k])
        return launch

    for k, b in enumerate(bands):
        streams[k].wait_event(ready[k])
        with torch.cuda.stream(streams[k]):
            _band_pieces(bufs[k], outs[k], b, wing, launcher(k), n_bands > 1, "interior")
    for k, b in enumerate(bands):
        with torch.cuda.stream(streams[k]):
            if b.above:
                up = bands[k - 1]
                streams[k].wait_event(ready[k - 1])
                bufs[k][:b.above].copy_(bufs[k - 1][up.above + up.rows - b.above:up.above + up.rows],
                                        non_blocking=True)
            if b.below:
                dn = bands[k + 1]
                streams[k].wait_event(ready[k + 1])
                bufs[k][b.above + b.rows:].copy_(bufs[k + 1][dn.above:dn.above + b.below], non_blocking=True)
            _band_pieces(bufs[k], outs[k], b, wing, launcher(k), n_bands > 1, "edges")
    for k, b in enumerate(bands):
        streams[k].synchronize()
        out[b.y0:b.y0 + b.rows].copy_(outs[k])
    torch.cuda.synchronize()
