#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_layout.py -q -p no:cacheprovider 2>&1 | tail -1
timeout 600 python bench.py --config 1 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 600 python bench.py --config 2 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
for c in 1 2; do python -c "
import json; d=json.loads(open('gpurun_out/bench_c$c.json').read().strip().splitlines()[-1]); L=d['layout']; print('c$c', d['value'], d['e2e']['value'], 'layout', L['value'], L['ms_total'])"; done
