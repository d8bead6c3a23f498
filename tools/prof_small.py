"""Per-phase cycles of the persistent small-mesh layout step (build the lib
with -DMDC_SMALL_PROF=1: tools/build_variant.sh smallprof ...).  Experiments only."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import load_golden  # noqa: E402
from helpers import golden_mesh  # noqa: E402
from paper_1408_0677_b200 import layout as L  # noqa: E402

for name in ("c1", "g2k"):
    g = load_golden(name)
    m = golden_mesh(g)
    p = L.LayoutParams.defaults_for(m, iterations=50)
    eng = L.LayoutEngine(m, p)
    temps = L.temperature_schedule(p.initial_temp, p.decay_lambda, 50)
    eng.set_positions(m.original_pos)
    eng.run(temps)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(7):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        eng.set_positions(m.original_pos)
        e0.record()
        eng.run(temps)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / 50)
    print(name, m.node_count, "us/step (best of 7)", best, flush=True)
