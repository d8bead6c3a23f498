#!/bin/bash
set -x
mkdir -p gpurun_out/bench_data
timeout 900 python tools/make_bench_positions.py && cp bench_data/config*_positions.npz gpurun_out/bench_data/
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
python -c "import json; d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['layout']['value'], d['layout']['positions_equal_cpu_arm_fixture'])"
