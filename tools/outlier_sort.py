"""Sort/tree robustness timing: repulsion (tree + BH) on 100k points whose
bulk is a tight cluster with a few far outliers, vs the same points without
the outliers.  Experiments only."""
import sys
import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1408_0677_b200 import bhtree  # noqa: E402

rng = np.random.default_rng(3)
n = 100_000
pts = rng.normal(0, 1.0, (n, 2))
out = pts.copy()
out[:4] = [[1e6, 0], [-1e6, 0], [0, 1e6], [0, -1e6]]
for name, p0 in (("gauss", pts), ("outliers", out)):
    p = torch.as_tensor(p0).cuda()
    f = bhtree.repulsive_forces_device(p, 1.0, 1e-3, 0.5)  # warm
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(5):
        f = bhtree.repulsive_forces_device(p, 1.0, 1e-3, 0.5)
    e1.record()
    torch.cuda.synchronize()
    print(name, "repulsive_forces ms", e0.elapsed_time(e1) / 5)
