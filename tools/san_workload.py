"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): every kernel family once at a size the tools finish quickly --
the tcgen05 MLS kernel (fp32 affine, d = 8 and d = 70: 16/64-channel chunks),
the SIMT MLS kernel (fp64 + fp32 mean/rigid), snap, fused band shading, the
layout step at n = 2000 (one-CTA / cluster walk), 20000 (cooperative grid walk
+ subtree CTAs + CUB sort) and the vertex-partitioned all-gather step, PCA,
render.  usage: compute-sanitizer --tool X python tools/san_workload.py"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_1408_0677_b200 import dataset as D  # noqa: E402
from paper_1408_0677_b200 import field as F  # noqa: E402
from paper_1408_0677_b200 import layout as L  # noqa: E402
from paper_1408_0677_b200 import mesh as M  # noqa: E402
from paper_1408_0677_b200 import projection as P  # noqa: E402
from paper_1408_0677_b200 import render as R  # noqa: E402

torch.cuda.set_device(0)
rng = np.random.default_rng(0)
X = bench.gmm(600, 70, 1)
ds = D.normalize(D.Dataset(names=[f"d{i}" for i in range(70)], data=X))
_, cloud = P.pca_project(ds)
pos = cloud.positions
raw = np.column_stack([ds.raw_column(nm) for nm in ds.names])
W, H = 64, 40
sp = np.full(70, 0.7)
for d in (8, 70):
    blk = F.compute_fields(pos, raw[:, :d], F.MlsParams("affine"), W, H, dtype="f32", band_spacing=sp[:d],
                           colormap=R.DEFAULT_COLORMAP)
    print("tc", d, float(blk.values.abs().max()))
for dt in ("f64", "f32"):
    for var in ("mean", "affine", "rigid"):
        blk = F.compute_fields(pos, raw[:, :2], F.MlsParams(var), W, H, dtype=dt, band_spacing=sp[:2],
                               tensor_cores=False)
        print(var, dt, float(blk.values.abs().max()))
for n in (2000, 20000):
    m = M.delaunay(bench.gmm(n, 2, 3), seed=0)
    params = L.LayoutParams.defaults_for(m, iterations=3)
    st = L.layout_run(m, params)
    print("layout", n, float(np.abs(st.relaxed_pos).max()))
torch.cuda.synchronize()
print("ok")
