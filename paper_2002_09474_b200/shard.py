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


def exchange_halos(buf, band: Band, world: int, rank: int, wing: int, dist=None, group=None) -> None:
    """Fill the halo rows of ``buf`` ([buffer_rows, W] tensor, band rows at [above, above+rows))
    from the neighbouring ranks: one batched point-to-point group (isend/irecv pairs).

    The rank above needs our first ``its below`` rows; the rank below needs our last ``its above``
    rows. Every band must hold at least ``wing`` rows (checked), so one hop suffices.
    """
    if dist is None:
        import torch.distributed as dist
    if band.rows == 0 or wing == 0 or world == 1:
        return
    per = -(-band.height // world)
    if per < wing:
        raise ValueError(f"bands of {per} rows are thinner than the halo ({wing}); use fewer ranks")
    up, down = neighbours(world, rank, band.height)
    ops = []
    a, r = band.above, band.rows
    if up is not None:
        ub = band_plan(band.height, world, up, wing)
        n_send = ub.below  # rows the rank above holds below its band = our first rows
        ops.append(dist.P2POp(dist.isend, buf[a:a + n_send].contiguous(), up, group))
        recv_up = buf.new_empty((a,) + tuple(buf.shape[1:]))
        ops.append(dist.P2POp(dist.irecv, recv_up, up, group))
    if down is not None:
        db = band_plan(band.height, world, down, wing)
        n_send = db.above  # rows the rank below holds above its band = our last rows
        ops.append(dist.P2POp(dist.isend, buf[a + r - n_send:a + r].contiguous(), down, group))
        recv_down = buf.new_empty((band.below,) + tuple(buf.shape[1:]))
        ops.append(dist.P2POp(dist.irecv, recv_down, down, group))
    if not ops:
        return
    for req in dist.batch_isend_irecv(ops):
        req.wait()
    if up is not None:
        buf[:a].copy_(recv_up)
    if down is not None:
        buf[a + r:].copy_(recv_down)


def morph_band(buf, out, band: Band, wx: int, wy: int, op: int, border: int = 0, value: int = 0,
               stream=None) -> None:
    """GPU compute of one band (``buf`` holds halo + band rows on the device, ``out`` the band rows)."""
    from .api import morph_band_device
    if band.rows == 0:
        return
    morph_band_device(buf, band.above, band.below, out, wx, wy, op, border, value, stream)
