#!/bin/bash
# A/B the SIMT MLS kernel (fp32): affine d=4 (SIMT by default), mean d=8, rigid d=2, affine d=32 --no-tc.
for L in "$@"; do
  MDC_LIB_PATH=$PWD/paper_1408_0677_b200/$L timeout 300 python - <<PY
import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
import bench
from paper_1408_0677_b200 import field as F
X = bench.gmm(100000, 32, 3)
pos = X[:, :2] * 3
for variant, d, tc in (("affine", 4, True), ("mean", 8, True), ("rigid", 2, True), ("affine", 32, False)):
    prob = F.MlsProblem(pos, X[:, :d], variant, 1920, 1080, dtype="f32", tensor_cores=tc)
    out = torch.empty((d, 1080, 1920), dtype=torch.float32, device="cuda")
    a = prob.args(out, (1080 * 1920, 1920, 1), 0, 1080)
    prob.run(a, snap=False); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); prob.run(a, snap=False); e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1)
    print("$L", variant, d, "tc" if tc else "simt", round(ms, 1), "ms", round(1920 * 1080 * d / ms / 1e3, 1), "Mpix*dim/s", flush=True)
PY
done
