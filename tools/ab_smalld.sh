#!/bin/bash
# A/B small-d fp32 affine: TC path (padded to 16 channels) vs SIMT kernel.
for D in 1 2 4 8; do for L in "$@"; do
  MDC_LIB_PATH=$PWD/paper_1408_0677_b200/$L timeout 300 python - <<PY
import sys, os, time, numpy as np, torch
sys.path.insert(0, os.getcwd())
import bench
from paper_1408_0677_b200 import field as F
X = bench.gmm(100000, $D, 3)
pos = np.column_stack([X[:, 0], X[:, -1] if $D > 1 else np.sin(X[:, 0] * 3)])
prob = F.MlsProblem(pos, X, "affine", 1920, 1080, dtype="f32")
out = torch.empty(($D, 1080, 1920), dtype=torch.float32, device="cuda")
a = prob.args(out, (1080 * 1920, 1920, 1), 0, 1080)
prob.run(a, snap=False); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); prob.run(a, snap=False); e1.record(); e1.synchronize()
ms = e0.elapsed_time(e1)
print("d=$D", "$L", round(ms, 1), "ms", round(1920 * 1080 * $D / ms / 1e3, 1), "Mpix*dim/s")
PY
done; done
