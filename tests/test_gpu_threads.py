"""Threading and determinism conventions of the boundary:
results are independent of the `threads` knob and of repetition
(test_field.py:251-261), and the library is reentrant from several Python
threads at once -- the service pattern (service.py:222-250) of a layout
running on a worker thread while requests render -- on one shared stream or
on a stream per thread."""
import threading

import numpy as np
import pytest
import torch

from conftest import layout_params
from helpers import golden_mesh
from paper_1408_0677_b200 import field as F
from paper_1408_0677_b200 import layout as L
from paper_1408_0677_b200 import mesh as M

pytestmark = pytest.mark.gpu


def test_compute_field_deterministic_and_thread_invariant():
    """test_field.py:251-261, every variant."""
    rng = np.random.default_rng(4)
    pts = rng.uniform(0, 5, (50, 2))
    mesh = M.delaunay(pts, seed=0)
    q = pts + rng.normal(0, 0.2, pts.shape)
    targets = F.TargetAssignment(targets=q, mode="projection")
    for variant in ("mean", "affine", "rigid", "linear"):
        params = F.MlsParams(variant=variant)
        a = F.compute_field(mesh, pts, targets, params, 64, 64, threads=1)
        b = F.compute_field(mesh, pts, targets, params, 64, 64, threads=1)
        c = F.compute_field(mesh, pts, targets, params, 64, 64, threads=4)
        assert a.coords.tobytes() == b.coords.tobytes() == c.coords.tobytes(), variant


def _mls_jobs():
    jobs = []
    for i, (n, d, W, H, dt) in enumerate(((3000, 16, 320, 200, "f32"), (500, 3, 128, 96, "f64"),
                                         (2000, 32, 256, 256, "f32"), (800, 2, 200, 150, "f64"))):
        rng = np.random.default_rng(40 + i)
        pos = rng.normal(0, 2.0, (n, 2))
        pos[:5] = pos[5:10]  # coincident controls: the snap scratch sees ties
        jobs.append((pos, rng.normal(0, 1.0, (n, d)), W, H, dt))
    return jobs


def _run_mls(job, stream=None):
    pos, q, W, H, dt = job
    ctx = torch.cuda.stream(stream) if stream is not None else torch.cuda.stream(torch.cuda.current_stream())
    with ctx:
        blk = F.compute_fields(pos, q, F.MlsParams("affine"), W, H, dtype=dt, band_spacing=np.full(q.shape[1], 0.25))
        vals, bands = blk.values.cpu().numpy(), blk.bands.cpu().numpy()
    return vals, bands


@pytest.mark.timeout(600)
@pytest.mark.parametrize("streams", ["shared", "per_thread"])
def test_concurrent_threads_match_sequential(g2k, streams):
    jobs = _mls_jobs()
    ref = [_run_mls(j) for j in jobs]
    m = golden_mesh(g2k)
    p = layout_params(g2k)
    lparams = L.LayoutParams(iterations=20, **{k: p[k] for k in (
        "repulsion_c", "spring_scale", "desired_edge_d", "softening_eta", "initial_temp", "decay_lambda",
        "bh_theta")})
    lay_ref = L.layout_run(m, lparams).relaxed_pos.copy()

    results, errors = {}, []

    def worker(key, fn):
        try:
            stream = torch.cuda.Stream() if streams == "per_thread" else None
            out = []
            for _ in range(3):
                out.append(fn(stream))
            results[key] = out
        except Exception as e:  # surfaced below
            errors.append((key, repr(e)))

    def layout_job(stream):
        ctx = torch.cuda.stream(stream) if stream is not None else torch.cuda.stream(torch.cuda.current_stream())
        with ctx:
            return L.layout_run(golden_mesh(g2k), lparams).relaxed_pos.copy()

    threads = [threading.Thread(target=worker, args=(("mls", i), lambda s, j=j: _run_mls(j, s)))
               for i, j in enumerate(jobs)]
    threads.append(threading.Thread(target=worker, args=(("layout", 0), layout_job)))
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for i in range(len(jobs)):
        for vals, bands in results[("mls", i)]:
            assert np.array_equal(vals, ref[i][0]), i
            assert np.array_equal(bands, ref[i][1]), i
    for pos in results[("layout", 0)]:
        assert np.array_equal(pos, lay_ref)
