"""Host overhead of the public API on a small frame (config 1: 256x256, N=150,
d=4): wall time of compute_fields_to_host split into its pieces, and a
cProfile of the call.  Experiments only."""
import cProfile
import pstats
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1408_0677_b200 import field as F  # noqa: E402
from paper_1408_0677_b200.render import DEFAULT_COLORMAP  # noqa: E402

W, H, n, d = 256, 256, 150, 4
rng = np.random.default_rng(1)
pos = torch.from_numpy(rng.normal(0, 3.0, (n, 2))).pin_memory()
raw = torch.from_numpy(rng.normal(0, 1.0, (n, d))).pin_memory()
out = torch.empty((d, H, W), dtype=torch.float32).pin_memory()
rgba = torch.empty((d, H, W, 4), dtype=torch.uint8).pin_memory()
sp = np.full(d, 0.25)


def call():
    F.compute_fields_to_host(pos, raw, F.MlsParams("affine"), W, H, out, band_spacing=sp, rgba_out=rgba,
                             colormap=DEFAULT_COLORMAP)


for _ in range(5):
    call()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(50):
    call()
t1 = time.perf_counter()
print(f"compute_fields_to_host: {1e6 * (t1 - t0) / 50:.0f} us/call -> {W * H * d / ((t1 - t0) / 50) / 1e6:.0f} Mpixel*dim/s")
t0 = time.perf_counter()
for _ in range(50):
    F.MlsProblem(pos, raw, "affine", W, H, dtype="f32")
torch.cuda.synchronize()
print(f"MlsProblem(): {1e6 * (time.perf_counter() - t0) / 50:.0f} us")
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    call()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
