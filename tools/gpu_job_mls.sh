#!/bin/bash
for L in ${LIBS:-libmdc.so}; do for rep in 1 2; do
MDC_LIB_PATH=$PWD/paper_1408_0677_b200/$L timeout 600 python bench.py --config 3 --no-cpu --no-e2e --no-fp64 --no-layout --steps ${STEPS:-3} --warmup 1 > /tmp/b.json 2>/dev/null
python -c "
import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print('$L', d['value'], d['ms_per_step'])"
done; done
for L in ${LIBS:-libmdc.so}; do
MDC_LIB_PATH=$PWD/paper_1408_0677_b200/$L timeout 900 python -m pytest tests/test_gpu_bench_parity.py tests/test_gpu_mls.py tests/test_gpu_parity_report.py -q -s -p no:cacheprovider 2>&1 | grep -E "passed|failed|worst|fp32" | sed "s/^/$L /" | head -12
done
