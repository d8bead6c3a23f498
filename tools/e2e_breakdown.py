"""Where the e2e frame time goes (experiments only): per-band kernel time
(CUDA events around MlsProblem.run) vs wall clock of compute_fields_to_host."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1408_0677_b200 import field as F  # noqa: E402

W, H, n, d = 3840, 2160, 100_000, 32
rng = np.random.default_rng(3)
pos = torch.from_numpy(rng.normal(0, 3.0, (n, 2))).pin_memory()
raw = torch.from_numpy(rng.normal(0, 1.0, (n, d))).pin_memory()
out = torch.empty((d, H, W), dtype=torch.float32).pin_memory()
evs = []
orig = F.MlsProblem.run


def run(self, a, snap=True):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    orig(self, a, snap)  # field kernel + snap
    e1.record()
    evs.append((a.row1 - a.row0, e0, e1))


F.MlsProblem.run = run
for rep in range(2):
    evs.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    F.compute_fields_to_host(pos, raw, F.MlsParams("affine"), W, H, out, band_spacing=np.full(d, 0.25))
    t1 = time.perf_counter()
    k = [(r, e0.elapsed_time(e1)) for r, e0, e1 in evs]
    print(f"wall {1e3 * (t1 - t0):.1f} ms; bands {[r for r, _ in k]}; kernel ms {[round(x, 1) for _, x in k]}; "
          f"sum {sum(x for _, x in k):.1f}; first band start -> last band end "
          f"{evs[0][1].elapsed_time(evs[-1][2]):.1f}")
