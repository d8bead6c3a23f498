"""Row-band MLS across ranks with the real kernels: two gloo
ranks sharing this box's GPU each compute their band of the frame through the
production path (MlsProblem: mdc_mls_field + mdc_mls_snap + fused bands) after
the per-frame control broadcast (shard.broadcast_controls), and
shard.gather_bands assembles the frame on rank 0.  It must be torch.equal to
the one-rank frame (values and band indices) -- the bit-identity the 8-GPU
run relies on.  Both the tcgen05 path (d = 8) and the SIMT path (d = 3)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

W, H, N = 200, 150, 3000


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _scene(d):
    import bench

    rng_data = bench.gmm(N, d, 7)
    rng = np.random.default_rng(8)
    pos = rng.normal(0, 1, (N, 2))
    spacing = np.linspace(0.5, 1.5, d)
    return pos, rng_data, spacing


def _frame(prob, d, r0, r1, spacing, dev):
    rows = r1 - r0
    out = torch.empty((d, rows, W), dtype=torch.float32, device=dev)
    bands = torch.empty((d, rows, W), dtype=torch.int32, device=dev)
    sp = torch.as_tensor(spacing).to(dev)
    a = prob.args(out, (rows * W, W, 1), r0, r1, bands, (rows * W, W), sp)
    prob.run(a, snap=True)
    return out, bands


def _worker(rank, world, port, d, out_dir):
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    sys.path.insert(0, os.path.dirname(here))
    import torch.distributed as dist

    from paper_1408_0677_b200.field import MlsProblem
    from paper_1408_0677_b200.shard import broadcast_controls, gather_bands, row_band

    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    pos, raw, spacing = _scene(d)
    prob = MlsProblem(pos, raw, "affine", W, H, dtype="f32")
    ctrl = [prob.pc_t, prob.q_t, prob.pm_t, prob.qm_t, prob.pos_t, prob.tvals_t]
    if rank != 0:  # prove the control block arrives by broadcast, not by recomputation
        for t in ctrl:
            t.zero_()
    broadcast_controls(ctrl, src=0)
    r0, r1 = row_band(rank, world, H)
    out, bands = _frame(prob, d, r0, r1, spacing, dev)
    full = gather_bands(out, H, dst=0)
    full_b = gather_bands(bands, H, dst=0)
    if rank == 0:
        torch.save({"values": full.cpu(), "bands": full_b.cpu()}, os.path.join(out_dir, f"ranks_{d}.pt"))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("d", [8, 3])
def test_two_rank_row_bands_equal_one_rank_frame(tmp_path, d):
    from paper_1408_0677_b200.field import MlsProblem

    mp.spawn(_worker, args=(2, _free_port(), d, str(tmp_path)), nprocs=2, join=True)
    got = torch.load(tmp_path / f"ranks_{d}.pt")
    pos, raw, spacing = _scene(d)
    prob = MlsProblem(pos, raw, "affine", W, H, dtype="f32")
    out, bands = _frame(prob, d, 0, H, spacing, torch.device("cuda", 0))
    assert torch.equal(got["values"], out.cpu())
    assert torch.equal(got["bands"], bands.cpu())
