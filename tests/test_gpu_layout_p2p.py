"""Vertex-partitioned layout with the peer-memory exchange:
two processes, each owning half the vertices, whose step kernels store their
slices straight into both processes' cudaIpc-mapped position buffers.  On
this single-GPU box both processes share the device; no kernel waits on
another process (steps are ordered by a host barrier), so this exercises the
exact code path an NVLink pair runs.  The trajectory must be bit-identical
to the single-process one, as must the all-gather (the default: packed owned
slices, all_gather_into_tensor, scatter through the step permutation) and
all-reduce exchanges."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, exchange, iters, out_dir):
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    sys.path.insert(0, os.path.dirname(here))
    import torch.distributed as dist

    from conftest import load_golden, layout_params
    from helpers import golden_mesh
    from paper_1408_0677_b200 import layout as L

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    g = load_golden("g2k")
    p = layout_params(g)
    params = L.LayoutParams(iterations=iters, **{k: p[k] for k in (
        "repulsion_c", "spring_scale", "desired_edge_d", "softening_eta", "initial_temp", "decay_lambda",
        "bh_theta")})
    st = L.layout_run_partitioned(golden_mesh(g), params, exchange=exchange)
    np.save(os.path.join(out_dir, f"{exchange}_{rank}.npy"), st.relaxed_pos)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("exchange", ["allgather", "p2p", "allreduce"])
def test_partitioned_exchange_bit_identical(tmp_path, g2k, exchange):
    from conftest import layout_params
    from helpers import golden_mesh
    from paper_1408_0677_b200 import layout as L

    iters = 5
    mp.spawn(_worker, args=(2, _free_port(), exchange, iters, str(tmp_path)), nprocs=2, join=True)
    p = layout_params(g2k)
    params = L.LayoutParams(iterations=iters, **{k: p[k] for k in (
        "repulsion_c", "spring_scale", "desired_edge_d", "softening_eta", "initial_temp", "decay_lambda",
        "bh_theta")})
    ref = L.layout_run(golden_mesh(g2k), params).relaxed_pos
    for r in range(2):
        got = np.load(tmp_path / f"{exchange}_{r}.npy")
        assert np.array_equal(got, ref), (exchange, r, np.abs(got - ref).max())


def _worker_1m(rank, world, port, mesh_path, iters, out_dir):
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    sys.path.insert(0, os.path.dirname(here))
    import torch.distributed as dist

    from helpers import golden_mesh
    from paper_1408_0677_b200 import layout as L

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    m = golden_mesh(np.load(mesh_path))
    params = L.LayoutParams.defaults_for(m, iterations=iters)
    st = L.layout_run_partitioned(m, params, exchange="allgather")
    np.save(os.path.join(out_dir, f"m1_{rank}.npy"), st.relaxed_pos)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(1200)
def test_partitioned_allgather_at_1m_vertices(tmp_path):
    """Config 4's layout size (1M Gaussian-mixture points, seed 4; Delaunay
    mesh): two processes, vertex-partitioned with the all-gather exchange,
    3 steps; bit-identical to one process."""
    import bench
    from helpers import golden_mesh
    from paper_1408_0677_b200 import layout as L
    from paper_1408_0677_b200 import mesh as M

    pts = bench.gmm(1_000_000, 2, 4)
    m = M.delaunay(pts, seed=0)
    path = tmp_path / "mesh1m.npz"
    np.savez(path, original_pos=m.original_pos, triangles=m.triangles, csr_offsets=m.csr_offsets,
             csr_targets=m.csr_targets, fan_offsets=m.fan_offsets, fan_nodes=m.fan_nodes)
    iters = 3
    mp.spawn(_worker_1m, args=(2, _free_port(), str(path), iters, str(tmp_path)), nprocs=2, join=True)
    g = np.load(path)
    mr = golden_mesh(g)
    ref = L.layout_run(mr, L.LayoutParams.defaults_for(mr, iterations=iters)).relaxed_pos
    for r in range(2):
        got = np.load(tmp_path / f"m1_{r}.npy")
        assert np.array_equal(got, ref), (r, np.abs(got - ref).max())
