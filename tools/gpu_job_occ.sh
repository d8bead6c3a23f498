#!/bin/bash
mkdir -p gpurun_out
for c in 2 3; do timeout 300 python bench.py --config $c --no-cpu --no-e2e --no-fp64 --steps 1 --warmup 1 > gpurun_out/b_c$c.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/b_c$c.json').read().strip().splitlines()[-1]); L=d['layout']; print('c$c', L['value'], json.dumps(L['roofline']['phases_ms_one_eager_step']))"; done
for L in libmdc.so libmdc_occ1.so libmdc_occ4.so; do
  for c in 2 3; do MDC_LIB_PATH=$PWD/paper_1408_0677_b200/$L timeout 300 python tools/prof_layout.py $c 2>&1 | grep graph | sed "s/^/$L c$c /"; done
done
