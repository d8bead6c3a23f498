"""Save the fused MLS outputs of the libmdc selected by MDC_LIB_PATH for a few
shapes (A/B bit-exactness of kernel variants; experiments only).
usage: MDC_LIB_PATH=... python tools/ab_bitexact.py out.npz"""
import sys

import numpy as np
import torch

from paper_1408_0677_b200 import field as F

cases = [(1920, 1080, 100_000, 32, None), (640, 480, 12_345, 40, None), (333, 217, 1001, 8, (17, 190)),
         (256, 256, 3, 16, None), (1000, 37, 50_001, 32, (5, 36))]
res = {}
for i, (W, H, n, d, rr) in enumerate(cases):
    rng = np.random.default_rng(i)
    pos = rng.normal(0, 3.0, (n, 2))
    q = rng.normal(0, 1.0, (n, d))
    for alpha in (1.5, 0.5):
        blk = F.compute_fields(pos, q, F.MlsParams("affine", alpha=alpha), W, H, dtype="f32", row_range=rr)
        res[f"c{i}_a{alpha}"] = blk.values.cpu().numpy()
torch.cuda.synchronize()
np.savez(sys.argv[1], **res)
print("saved", len(res))
