"""Multi-process (gloo, CPU) tests of the N>1 host logic: the row-band plan of libgc
(gc_band_plan) and the halo exchange it prescribes, checked against the oracle, and the
batch sharding used by bench.py for c4.  No GPU: the halo rows travel over gloo
send/recv here, over NCCL inside gc_bilateral_band on the GPU box.
"""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _band_worker(rank, world, port, H, W, sigma_s, sigma_r, N, band_rows, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import paper_1605_02178_b200 as gc
        from synth import config_image
        full = config_image("c5", H=H, W=W)             # every rank can regenerate; it keeps only its band
        pl = gc.band_plan(H, rank, world, band_rows, sigma_s)
        r0, hb = pl["row0"], band_rows[rank]
        band = torch.from_numpy(np.ascontiguousarray(full[r0:r0 + hb]))
        R = math.ceil(3 * sigma_s)
        # exchange exactly what gc_bilateral_band exchanges: first R rows up, last R rows down
        top = torch.empty((pl["top_rows"], W)) if pl["top_rows"] else None
        bot = torch.empty((pl["bot_rows"], W)) if pl["bot_rows"] else None
        reqs = []
        if rank > 0:
            reqs.append(dist.isend(band[:R].contiguous(), rank - 1))
            reqs.append(dist.irecv(top, rank - 1))
        if rank < world - 1:
            reqs.append(dist.isend(band[hb - R:].contiguous(), rank + 1))
            reqs.append(dist.irecv(bot, rank + 1))
        for r in reqs:
            r.wait()
        # assemble what this rank holds into a global-shaped array; rows it does not hold are NaN
        g = np.full((H, W), np.nan, np.float32)
        g[r0:r0 + hb] = band.numpy()
        if top is not None:
            g[pl["top0"]:pl["top0"] + pl["top_rows"]] = top.numpy()
        if bot is not None:
            g[pl["bot0"]:pl["bot0"] + pl["bot_rows"]] = bot.numpy()
        rows = list(range(r0, r0 + hb))
        mine, _ = oracle.gc_filter_rows(g, rows, sigma_s, sigma_r, N)
        ref, _ = oracle.gc_filter_rows(full, rows, sigma_s, sigma_r, N)
        q.put((rank, float(np.nanmax(np.abs(mine - ref))), bool(np.all(np.isfinite(mine)))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,band_rows", [(2, [60, 57]), (3, [40, 40, 37]), (4, [30, 29, 29, 29])])
def test_band_halo_exchange_matches_whole_image(world, band_rows):
    H, W, sigma_s, sigma_r, N = sum(band_rows), 48, 3.0, 55.0, 12
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_band_worker, args=(r, world, port, H, W, sigma_s, sigma_r, N, band_rows, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, err, finite in res:
        assert finite, rank                       # every row the window needs was present
        assert err == 0.0, (rank, err)            # identical sums -> identical result


def _shard_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        B = 256
        per = B // world
        mine = torch.arange(rank * per, (rank + 1) * per, dtype=torch.int64)   # bench.py's c4 split
        out = [torch.empty(per, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(out, mine)
        allv = torch.cat(out)
        t = torch.tensor([float(rank + 1)])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)                                 # max-over-ranks timing
        q.put((rank, sorted(allv.tolist()) == list(range(B)), float(t.item())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_batch_shard_covers_every_image_once(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok, _ in res)
    assert all(mx == float(world) for _, _, mx in res)
