"""100k GMM points, 3840x2160, affine fp32, d in
{4, 8, ..., 256} -- Mpixel*dim/s and the FP32-lane roofline fraction of the
MLS kernel per d (device-resident, CUDA-event timed, L2 flushed)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1408_0677_b200 import _lib  # noqa: E402
from paper_1408_0677_b200 import field as F  # noqa: E402
from paper_1408_0677_b200 import projection as P  # noqa: E402
from paper_1408_0677_b200 import dataset as D  # noqa: E402


def main():
    lib = _lib.require_cuda()
    peaks = bench.measure_peaks(lib, torch)
    W, H, n = 3840, 2160, 100_000
    X = bench.gmm(n, 256, 3)
    ds = D.normalize(D.Dataset(names=[f"d{i}" for i in range(256)], data=X))
    _, cloud = P.pca_project(ds)
    raw = np.column_stack([ds.raw_column(nm) for nm in ds.names])
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    rows = []
    for d in (4, 8, 16, 32, 64, 128, 256):
        prob = F.MlsProblem(cloud.positions, raw[:, :d], "affine", W, H, dtype="f32")
        out = torch.empty((d, H, W), dtype=torch.float32, device="cuda")
        a = prob.args(out, (H * W, W, 1), 0, H)
        prob.run(a, snap=False)
        flush.fill_(1)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        prob.run(a, snap=False)
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        pairs = W * H * n
        if d >= 8:
            nc = 16 if d <= 16 else (32 if d <= 32 else (64 if d <= 64 else 128))  # mls_tc.cu pick_nc
            chunks = -(-d // nc)
            lane_ops, path = 13 + 10 * chunks, "tcgen05"  # pass 1: 13 (alpha = 3/2, sum 1/r)
        else:
            lane_ops, path = 14 + 9 + d, "simt"  # DC = d here (one chunk)
        frac = 2 * pairs * lane_ops / (ms * 1e-3) / peaks["fp32"]
        rows.append({"d": d, "path": path, "ms": ms, "mpix_dim_per_s": W * H * d / ms / 1e3,
                     "fp32_lane_frac": frac})
        print(json.dumps(rows[-1]), flush=True)
        del out, prob
        torch.cuda.empty_cache()
    print(json.dumps({"sweep": "config5", "frame": [W, H], "n": n, "rows": rows}))


if __name__ == "__main__":
    main()
