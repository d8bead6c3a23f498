"""One fp64 MLS launch (mls_kernel<double>, the parity mode) on a 16-row band
of the config-3 frame (PCA positions), for ncu: executed fp64 lane-ops per
(pixel, control) pair -> profiles/r02_mls_fp64_ops.json (bench.py's fp64
roofline).  usage: ncu ... python tools/prof_fp64.py"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_1408_0677_b200 import dataset as D  # noqa: E402
from paper_1408_0677_b200 import field as F  # noqa: E402
from paper_1408_0677_b200 import projection as P  # noqa: E402

cfg = bench.CONFIGS[3]
X = bench.gmm(cfg["n"], cfg["d"], cfg["seed"])
ds = D.normalize(D.Dataset(names=[f"d{i}" for i in range(cfg["d"])], data=X))
_, cloud = P.pca_project(ds)
raw = np.column_stack([ds.raw_column(nm) for nm in ds.names])
W, H, rows = cfg["W"], cfg["H"], int(os.environ.get("MDC_PROF_ROWS", "16"))
prob = F.MlsProblem(cloud.positions, raw, "affine", W, H, dtype="f64")
out = torch.empty((cfg["d"], rows, W), dtype=torch.float64, device="cuda")
a = prob.args(out, (rows * W, W, 1), H // 2, H // 2 + rows)
prob.run(a, snap=False)
torch.cuda.synchronize()
print("pairs", rows * W * cfg["n"])
