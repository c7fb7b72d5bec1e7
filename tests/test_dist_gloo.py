"""Multi-process (gloo, CPU) tests of the N>1 host logic, exercising the repo's own code:
libgc's row-band plan (gc_band_plan) and exchange plan (gc_band_exchange_plan: the peers,
offsets and counts gc_filter_band hands to ncclSend/ncclRecv) executed over gloo and checked
against the oracle on the whole image, and bench.py's c4 batch sharding (shard_of) and c5
band split (band_rows_of).  No GPU: the halo rows travel over gloo here, over NCCL inside
gc_filter_band on the GPU box.
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
        pl = gc.band_plan(H, rank, world, band_rows, sigma_s)
        r0, hb = pl["row0"], band_rows[rank]
        band = torch.from_numpy(config_image("c5", H=H, W=W, rows=(r0, r0 + hb)))   # only this rank's rows
        # execute libgc's own exchange plan (gc_band_exchange_plan: the offsets, counts and peers
        # gc_filter_band hands to ncclSend/ncclRecv) over gloo instead of NCCL
        xfers, segs = gc.band_exchange_plan(hb, W, H, r0, rank, world, sigma_s)
        flat = band.reshape(-1)
        recv, reqs = [None, None], []
        for k, x in enumerate(xfers):
            if x["peer"] < 0:
                continue
            recv[k] = torch.empty(x["count"])
            reqs.append(dist.isend(flat[x["send_offset"]:x["send_offset"] + x["count"]].contiguous(), x["peer"]))
            reqs.append(dist.irecv(recv[k], x["peer"]))
        for r in reqs:
            r.wait()
        # assemble the three segments gc_filter_window would read into a global-shaped array;
        # rows no segment holds stay NaN (an incomplete plan shows up as non-finite output)
        g = np.full((H, W), np.nan, np.float32)
        seg_data = [recv[0], band.reshape(-1), recv[1]]
        for (s0, sn), d in zip(segs, seg_data):
            if sn:
                g[s0:s0 + sn] = d.numpy().reshape(sn, W)
        assert pl["top_rows"] == segs[0][1] and pl["bot_rows"] == segs[2][1]
        rows = list(range(r0, r0 + hb))
        mine, _ = oracle.gc_filter_rows(g, rows, sigma_s, sigma_r, N)
        full = config_image("c5", H=H, W=W)
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


def test_c5_band_split_covers_the_image():
    """bench.py's c5 split over 1..8 ranks: contiguous bands, sizes within one row, every band
    accepted by libgc's plan (H_band > W_s)."""
    import sys
    sys.path.insert(0, ROOT)
    import bench
    import paper_1605_02178_b200 as gc
    for ws in range(1, 9):
        rows = bench.band_rows_of(16384, ws)
        assert sum(rows) == 16384 and max(rows) - min(rows) <= 1
        for r in range(ws):
            gc.band_plan(16384, r, ws, rows, 16.0)


def _shard_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        B = 256
        mine = torch.tensor(bench.shard_of(B, world, rank), dtype=torch.int64)   # bench.py's c4 split
        n = torch.tensor([len(mine)])
        sizes = [torch.empty(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(sizes, n)
        mx = int(max(v.item() for v in sizes))
        pad = torch.full((mx,), -1, dtype=torch.int64)
        pad[:len(mine)] = mine
        out = [torch.empty(mx, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(out, pad)
        allv = torch.cat(out)
        allv = allv[allv >= 0]
        t = torch.tensor([float(rank + 1)])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)                                 # max-over-ranks timing
        q.put((rank, sorted(allv.tolist()) == list(range(B)) and len(allv) == B, float(t.item())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3, 4])
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
