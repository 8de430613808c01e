"""Host logic of the multi-GPU sharding (paper_2002_09474_b200/shard.py) on CPU with the gloo
backend, world size 2: batch shards, row-band plans, and the halo exchange. The per-band compute is
stood in for by the oracle on the local buffer (the product computes it with rmgpu_morph_band_* on the
GPU; tests/test_gpu_parity.py::test_row_bands covers that kernel path)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2002_09474_b200.shard import (_band_pieces, band_plan, batch_shard, exchange_halos, interior_rows,
                                          neighbours, start_halo_exchange)


def test_batch_shard_covers_everything():
    for n in (0, 1, 7, 512, 513):
        for g in (1, 2, 3, 4, 8):
            got = [batch_shard(n, g, r) for r in range(g)]
            assert sum(c for _, c in got) == n
            assert all(got[i][0] + got[i][1] == got[i + 1][0] for i in range(g - 1))
            assert max(c for _, c in got) - min(c for _, c in got) <= 1


def test_band_plan_partitions_rows():
    for h in (1, 62, 100, 4096, 32768):
        for g in (1, 2, 4, 8):
            for wing in (0, 1, 31):
                bands = [band_plan(h, g, r, wing) for r in range(g)]
                assert sum(b.rows for b in bands) == h
                y = 0
                for b in bands:
                    assert b.y0 == y or b.rows == 0
                    y += b.rows
                    assert b.above == min(wing, b.y0)
                    assert b.below == min(wing, h - b.y0 - b.rows)
    assert neighbours(4, 0, 100) == (None, 1)
    assert neighbours(4, 3, 100) == (2, None)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, h, w, wx, wy, op, border, bval, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        R = oracle.restatement()
        full = R.generate(w, h, 55)
        wing = wy // 2
        band = band_plan(h, world, rank, wing)
        # local buffer: band rows from "our memory", halo rows poisoned until the exchange
        buf = torch.full((band.buffer_rows, w), 0xEE, dtype=torch.uint8)
        buf[band.above:band.above + band.rows] = torch.from_numpy(full[band.y0:band.y0 + band.rows])
        # the overlapped schedule of morph_band_overlapped: issue the exchange (received straight
        # into the poisoned halo rows), compute the interior pieces while it is in flight, wait,
        # compute the edge pieces. The oracle on the piece's rows stands in for rmgpu_morph_band_u8
        # (same semantics: the piece's first / last context rows are its border); an interior piece
        # that read a halo row would see poison or a racing receive and differ.
        out = torch.zeros((band.rows, w), dtype=torch.uint8)

        def launch(src, above, below, dst):
            n = dst.shape[0]
            local = R.morph(np.ascontiguousarray(src[:above + n + below].numpy()), wx, wy, op, border, bval)
            dst.copy_(torch.from_numpy(np.ascontiguousarray(local[above:above + n])))

        reqs = start_halo_exchange(buf, band, world, rank, wing, dist=dist)
        _band_pieces(buf, out, band, wing, launch, bool(reqs), "interior")
        for req in reqs:
            req.wait()
        _band_pieces(buf, out, band, wing, launch, bool(reqs), "edges")
        want_buf = full[band.in_y0:band.in_y0 + band.buffer_rows]
        ok_exchange = bool(np.array_equal(buf.numpy(), want_buf))
        mine = out
        sizes = [band_plan(h, world, r, wing).rows for r in range(world)]
        parts = [torch.empty((s, w), dtype=torch.uint8) for s in sizes]
        dist.all_gather(parts, mine) if len(set(sizes)) == 1 else _gather_ragged(parts, mine, rank, world)
        if rank == 0:
            whole = torch.cat(parts).numpy()
            q.put((ok_exchange, bool(np.array_equal(whole, R.morph(full, wx, wy, op, border, bval)))))
        else:
            q.put((ok_exchange, True))
    finally:
        dist.destroy_process_group()


def _gather_ragged(parts, mine, rank, world):
    for r in range(world):
        if r == rank:
            parts[r].copy_(mine)
        dist.broadcast(parts[r], src=r)


@pytest.mark.parametrize("h,wx,wy,op,border,bval", [(64, 3, 3, 0, 0, 0), (101, 5, 31, 1, 0, 0), (77, 7, 21, 0, 1, 9),
                                                     (62, 1, 61, 1, 0, 0), (200, 9, 15, 4, 0, 0), (90, 3, 29, 4, 1, 77)])
def test_row_bands_gloo_world2(h, wx, wy, op, border, bval):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, h, 45, wx, wy, op, border, bval, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(r[0] for r in res), "halo exchange delivered wrong rows"
    assert all(r[1] for r in res), "banded result differs from the whole-image oracle"


def test_band_pieces_cover_the_band_single_process():
    # the interior / edge decomposition of morph_band_overlapped, every band of several splits:
    # the interior pieces never read a halo row (poisoned until "arrival"), edges + interior
    # reproduce the whole-image result exactly
    import oracle
    R = oracle.restatement()
    for h, w, wy, nb in ((97, 33, 11, 3), (64, 20, 31, 2), (300, 17, 21, 5), (40, 9, 3, 8)):
        full = R.generate(w, h, h + wy)
        want = R.morph(full, 5, wy, 1)
        wing = wy // 2
        got = np.zeros_like(full)
        for k in range(nb):
            band = band_plan(h, nb, k, wing)
            if band.rows == 0:
                continue
            buf = torch.full((band.buffer_rows, w), 0xEE, dtype=torch.uint8)
            buf[band.above:band.above + band.rows] = torch.from_numpy(full[band.y0:band.y0 + band.rows])
            out = torch.zeros((band.rows, w), dtype=torch.uint8)

            def launch(src, above, below, dst):
                n = dst.shape[0]
                local = R.morph(np.ascontiguousarray(src[:above + n + below].numpy()), 5, wy, 1)
                dst.copy_(torch.from_numpy(np.ascontiguousarray(local[above:above + n])))

            pending = band.above > 0 or band.below > 0
            _band_pieces(buf, out, band, wing, launch, pending, "interior")
            lo, hi = interior_rows(band, wing)
            if pending:  # halos arrive
                buf[:] = torch.from_numpy(full[band.in_y0:band.in_y0 + band.buffer_rows])
            _band_pieces(buf, out, band, wing, launch, pending, "edges")
            got[band.y0:band.y0 + band.rows] = out.numpy()
        assert np.array_equal(got, want), (h, w, wy, nb)
