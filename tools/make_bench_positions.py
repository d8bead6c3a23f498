"""Write bench_data/config{2,3}_positions.npz: the GPU layout's positions
after 250 and `iters` iterations, exactly as bench.py computes them (same
scene, same CUDA-graph steps).  The CPU arm times the reference's MLS at the
laid-out positions and the reference's layout step from iterations 0 and 250
from these; bench.py's GPU arm checks its own final positions
equal the file.  Run on the GPU box: python tools/make_bench_positions.py"""
import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_1408_0677_b200 import layout as L  # noqa: E402


def main(ids):
    for cid in ids:
        cfg = dict(bench.CONFIGS[cid], id=cid)
        ds, mesh, raw = bench.build_scene(cfg)
        params = L.LayoutParams.defaults_for(mesh, iterations=cfg["iters"])
        temps = L.temperature_schedule(params.initial_temp, params.decay_lambda, cfg["iters"])
        eng = L.LayoutEngine(mesh, params)
        eng.set_positions(mesh.original_pos)
        eng.run(temps)  # bench.py's warm-up + capture
        eng.set_positions(mesh.original_pos)
        eng.run(temps[:250])
        p250 = eng.pos.cpu().numpy()
        eng.run(temps[250:])
        pfin = eng.pos.cpu().numpy()
        eng2 = L.LayoutEngine(mesh, params)
        eng2.set_positions(mesh.original_pos)
        eng2.run(temps)
        assert np.array_equal(eng2.pos.cpu().numpy(), pfin), "the split run must equal bench.py's one-call run"
        path = os.path.join(ROOT, "bench_data", f"config{cid}_positions.npz")
        tri = np.ascontiguousarray(mesh.triangles.astype(np.int64))
        np.savez_compressed(path, iters=np.int64(cfg["iters"]), original_pos=mesh.original_pos,
                            triangles_sha256=np.array(hashlib.sha256(tri.tobytes()).hexdigest()),
                            pos_250=p250, pos_final=pfin)
        print("wrote", path, os.path.getsize(path))


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [2, 3])
