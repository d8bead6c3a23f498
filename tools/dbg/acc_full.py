"""Accuracy of the fp32 MLS paths at the bench's full size (config 3) on a few row bands vs the fp64 oracle."""
import sys, os, time, numpy as np
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "oracle"))
import oracle as O
import bench
from paper_1408_0677_b200 import field as F
cfg = dict(bench.CONFIGS[int(os.environ.get("CFG", "3"))], id=3)
ds, mesh, raw = bench.build_scene(cfg)
pos = mesh.original_pos
W, H = cfg["W"], cfg["H"]
bands = [(0, 8), (H // 2 - 4, H // 2 + 4), (H - 8, H)]
chans = [0, 16, 31] if raw.shape[1] > 31 else [0, raw.shape[1] - 1]
for tag, kw in (("tc", {}), ("simt", {"tensor_cores": False})):
    if tag == "simt" and os.environ.get("NO_SIMT"):
        continue
    errs = []
    for (r0, r1) in bands:
        v = F.compute_fields(pos, raw, F.MlsParams("affine"), W, H, dtype="f32", row_range=(r0, r1), **kw).values.double().cpu().numpy()
        for i in range(0, len(chans), 2):
            cs = chans[i:i + 2] if i + 1 < len(chans) else [chans[i], chans[i]]
            t0 = time.time()
            ref = O.compute_field(pos, raw[:, cs], "affine", W, H, rows=(r0, r1))
            for j, c in enumerate(cs):
                e = np.abs(v[c] - ref[..., j]).max() / np.abs(ref[..., j]).max()
                errs.append(e)
                print(tag, (r0, r1), c, f"{e:.3e}", f"oracle {time.time() - t0:.1f}s", flush=True)
    print(tag, "max normwise", max(errs))
