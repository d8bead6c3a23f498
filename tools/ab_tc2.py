"""A/B of the one-pass (mls_tc2) vs the two-pass (mls_tc) tensor-core MLS
kernel on a bench-shaped frame: CUDA-event time of each, and the fp32 error
of each against the fp64 oracle on a few rows (all channels).  Experiments
only (not a test, not the bench).

usage: python tools/ab_tc2.py [WxH] [n] [d] [rows...]
"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import bench  # noqa: E402
import oracle as O  # noqa: E402
from paper_1408_0677_b200 import _lib  # noqa: E402
from paper_1408_0677_b200 import dataset as D  # noqa: E402
from paper_1408_0677_b200 import field as F  # noqa: E402
from paper_1408_0677_b200 import projection as P  # noqa: E402


def P_pix(pos, W, H):
    vp = O.viewport(pos, W, H)
    x0, y0, x1, y1, sx, sy = vp
    return np.column_stack([(pos[:, 0] - x0) / sx, (y1 - pos[:, 1]) / sy])


def main():
    wh = sys.argv[1] if len(sys.argv) > 1 else "1920x1080"
    W, H = (int(v) for v in wh.split("x"))
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 100_000
    d = int(sys.argv[3]) if len(sys.argv) > 3 else 32
    rows = [int(r) for r in sys.argv[4:]] or [0, H // 3, H // 2, H - 1]
    alpha = float(os.environ.get("AB_ALPHA", "1.5"))
    X = bench.gmm(n, d, 3)
    ds = D.normalize(D.Dataset(names=[f"d{i}" for i in range(d)], data=X))
    _, cloud = P.pca_project(ds)
    pos = cloud.positions
    raw = np.column_stack([ds.raw_column(nm) for nm in ds.names])
    t0 = time.time()
    ref = O.affine_fields(pos, raw, W, H, rows=rows, alpha=alpha)
    print(f"oracle {len(rows)} rows x {d} ch: {time.time() - t0:.1f} s", flush=True)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    outs = {}
    only = os.environ.get("AB_ONLY")
    variants = [v for v in (("onepass", _lib.MDC_FLAG_TC_ONEPASS), ("twopass", 0)) if only in (None, v[0])]
    if os.environ.get("AB_NOREF"):
        ref = None
    for name, flags in variants:
        prob = F.MlsProblem(pos, raw, "affine", W, H, alpha=alpha, dtype="f32")
        prob.flags = flags
        out = torch.empty((d, H, W), dtype=torch.float32, device="cuda")
        a = prob.args(out, (H * W, W, 1), 0, H)
        prob.run(a, snap=False)
        torch.cuda.synchronize()
        ms = []
        for _ in range(3):
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            prob.run(a, snap=False)
            e1.record()
            e1.synchronize()
            ms.append(e0.elapsed_time(e1))
        v = out[:, rows, :].double().cpu().numpy().transpose(1, 2, 0)
        err = -1.0 if ref is None else max(np.abs(v[..., k] - ref[..., k]).max() / np.abs(ref[..., k]).max()
                                           for k in range(d))
        if ref is not None:
            e = np.abs(v - ref)
            i = np.unravel_index(np.argmax(e), e.shape)
            print(f"  worst vs oracle at row {rows[i[0]]} col {i[1]} ch {i[2]}: got {v[i]:.6f} ref {ref[i]:.6f}")
        outs[name] = out
        print(f"{name}: {min(ms):.2f} ms  {W * H * d / min(ms) / 1e3:.1f} Mpixel*dim/s  "
              f"normwise err vs oracle {err:.3e}  finite={bool(torch.isfinite(out).all())}", flush=True)
    if len(outs) == 2:
        dd = (outs["onepass"] - outs["twopass"]).abs()
        diff = dd.max().item()
        i = np.unravel_index(int(dd.argmax()), dd.shape)
        print(f"max |onepass - twopass| = {diff:.3e} at ch {i[0]} row {i[1]} col {i[2]} "
              f"(one {outs['onepass'][i].item():.5f} two {outs['twopass'][i].item():.5f}); "
              f"pixels > 1e-3: {int((dd.amax(0) > 1e-3).sum())}")
        ctl = P_pix(pos, W, H)
        dist = np.sqrt(((ctl - np.array([i[2] + 0.5, i[1] + 0.5])) ** 2).sum(1)).min()
        print(f"  nearest control to that pixel: {dist:.3f} px")


if __name__ == "__main__":
    main()
