"""Multi-process (world_size 2, gloo, CPU) test of the row-band sharding host
logic used for N-GPU MLS frames: band partition, per-frame control-block
broadcast, band gather == single-rank frame."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1408_0677_b200.shard import broadcast_controls, gather_bands, row_band


def test_row_bands_partition_rows():
    for world in (1, 2, 3, 4, 8):
        for h in (1, 7, 48, 2160):
            if h < world:
                continue
            bands = [row_band(r, world, h) for r in range(world)]
            assert bands[0][0] == 0 and bands[-1][1] == h
            assert all(a[1] == b[0] for a, b in zip(bands, bands[1:]))
            sizes = [r1 - r0 for r0, r1 in bands]
            assert max(sizes) - min(sizes) <= 1


def _frame(h, w, d):
    # stand-in for a field: a deterministic function of the global pixel index
    idx = torch.arange(h * w, dtype=torch.float64).reshape(1, h, w)
    return torch.cat([idx * (k + 1) for k in range(d)], dim=0)


def _worker(rank, world, port, h, w, d, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ctrl = [torch.arange(12, dtype=torch.float64) if rank == 0 else torch.zeros(12, dtype=torch.float64),
                torch.full((5, 3), 7.0) if rank == 0 else torch.zeros(5, 3)]
        broadcast_controls(ctrl, src=0)
        ok_bcast = torch.equal(ctrl[0], torch.arange(12, dtype=torch.float64)) and bool((ctrl[1] == 7).all())
        r0, r1 = row_band(rank, world, h)
        local = _frame(h, w, d)[:, r0:r1].contiguous()
        full = gather_bands(local, h, dst=0)
        ok_gather = True if rank != 0 else torch.equal(full, _frame(h, w, d))
        q.put((rank, ok_bcast, ok_gather))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,h", [(2, 9), (2, 48)])
def test_gloo_broadcast_and_gather(world, h):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, h, 5, 3, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok_b and ok_g for _, ok_b, ok_g in res), res
