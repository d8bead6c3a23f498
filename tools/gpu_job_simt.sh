#!/bin/bash
for L in ${LIBS:-libmdc.so}; do
  MDC_LIB_PATH=$PWD/paper_1408_0677_b200/$L timeout 600 python bench.py --config 3 --no-cpu --no-e2e --no-layout --steps 1 --warmup 1 > /tmp/b.json 2>/dev/null
  python -c "
import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); f=d['fp64']; print('$L fp64', f['value'], f['kernel_ms'])"
  MDC_LIB_PATH=$PWD/paper_1408_0677_b200/$L timeout 600 python bench.py --config 1 --no-cpu --no-e2e --no-layout --no-fp64 --steps 20 --warmup 3 > /tmp/b1.json 2>/dev/null
  python -c "
import json; d=json.loads(open('/tmp/b1.json').read().strip().splitlines()[-1]); print('$L c1', d['value'], d['ms_per_step'])"
  MDC_LIB_PATH=$PWD/paper_1408_0677_b200/$L timeout 900 python -m pytest tests/test_gpu_mls.py tests/test_gpu_bench_parity.py tests/test_gpu_closed_form.py tests/test_gpu_render.py -q -s -p no:cacheprovider 2>&1 | grep -E "passed|failed|worst|normwise" | sed "s/^/$L /" | head -12
done
