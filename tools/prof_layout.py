import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import bench
from paper_1408_0677_b200 import layout as L, _lib
cfg = dict(bench.CONFIGS[int(sys.argv[1])], id=int(sys.argv[1]))
ds, mesh, raw = bench.build_scene(cfg)
params = L.LayoutParams.defaults_for(mesh, iterations=50)
eng = L.LayoutEngine(mesh, params)
temps = L.temperature_schedule(params.initial_temp, params.decay_lambda, 50)
pos0 = torch.as_tensor(mesh.original_pos).cuda()
def t(fn, reps=20):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1000
out = torch.empty_like(pos0)
h = eng.plan()
lib = eng.lib
print("repulsion (tree+BH) us", t(lambda: lib.mdc_layout_repulsion(h, _lib.ptr(pos0), _lib.ptr(out), _lib.stream_ptr())))
eng.set_positions(mesh.original_pos)
print("step eager us", t(lambda: eng.run(temps[:1], use_graph=False)))
print("step graph x50 us/step", t(lambda: eng.run(temps, use_graph=True), reps=3) / 50)
