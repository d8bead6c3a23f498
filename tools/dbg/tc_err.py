import sys, os, numpy as np
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "oracle"))
import oracle as O
from paper_1408_0677_b200 import field as F
for (n, d, W, H, alpha) in [(2000, 8, 96, 64, 1.5), (150, 8, 64, 48, 1.5), (2000, 8, 96, 64, 1.0), (600, 8, 96, 64, 1.5)]:
    rng = np.random.default_rng(n + d)
    pos = rng.normal(0, 3, (n, 2))
    q = rng.normal(0, 1, (n, d)) + pos[:, :1] * np.arange(d)
    tc = F.compute_fields(pos, q, F.MlsParams("affine", alpha=alpha), W, H, dtype="f32").values.double().cpu().numpy()
    si = F.compute_fields(pos, q, F.MlsParams("affine", alpha=alpha), W, H, dtype="f32", tensor_cores=False).values.double().cpu().numpy()
    k = 2
    ref = O.compute_field(pos, np.column_stack([q[:, k], np.zeros(n)]), "affine", W, H, alpha=alpha)[..., 0]
    e_tc = np.abs(tc[k] - ref); e_si = np.abs(si[k] - ref)
    print(n, d, W, H, alpha, "tc", e_tc.max() / np.abs(ref).max(), "simt", e_si.max() / np.abs(ref).max())
    r, c = np.unravel_index(np.argmax(e_tc), e_tc.shape)
    print("  worst px", r, c, tc[k][r, c], ref[r, c], "rows with err>1e-4:", sorted(set(np.nonzero(e_tc > 1e-4 * np.abs(ref).max())[0].tolist()))[:20])
