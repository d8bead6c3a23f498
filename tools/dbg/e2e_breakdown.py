import sys, os, time, numpy as np, torch
sys.path.insert(0, os.getcwd())
import bench
from paper_1408_0677_b200 import field as F
cfg = dict(bench.CONFIGS[3], id=3)
ds, mesh, raw = bench.build_scene(cfg)
pos = mesh.original_pos
W, H, d = cfg["W"], cfg["H"], cfg["d"]
sp = np.array([bench._auto_spacing(raw[:, k]) for k in range(d)])
pin_pos = torch.from_numpy(np.ascontiguousarray(pos)).pin_memory()
pin_raw = torch.from_numpy(np.ascontiguousarray(raw)).pin_memory()
host = torch.empty((d, H, W), dtype=torch.float32).pin_memory()
mp = F.MlsParams("affine")
for nb in (1, 4, 8, 16):
    F.compute_fields_to_host(pin_pos, pin_raw, mp, W, H, host, dtype="f32", band_spacing=sp, nbands=nb)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(2):
        F.compute_fields_to_host(pin_pos, pin_raw, mp, W, H, host, dtype="f32", band_spacing=sp, nbands=nb)
    t1 = time.perf_counter()
    print("nbands", nb, "ms", (t1 - t0) / 2 * 1e3, flush=True)
t0 = time.perf_counter()
for _ in range(3):
    prob = F.MlsProblem(pin_pos, pin_raw, "affine", W, H, dtype="f32")
torch.cuda.synchronize()
print("MlsProblem ms", (time.perf_counter() - t0) / 3 * 1e3)
out = torch.empty((d, H, W), dtype=torch.float32, device="cuda")
a = prob.args(out, (H * W, W, 1), 0, H)
prob.run(a); torch.cuda.synchronize()
t0 = time.perf_counter(); prob.run(a); torch.cuda.synchronize(); print("run (mls+snap) ms", (time.perf_counter() - t0) * 1e3)
t0 = time.perf_counter(); host.copy_(out, non_blocking=True); torch.cuda.synchronize(); print("D2H 1.06GB ms", (time.perf_counter() - t0) * 1e3)
