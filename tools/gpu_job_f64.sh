#!/bin/bash
for L in ${LIBS:-libmdc.so}; do
  MDC_LIB_PATH=$PWD/paper_1408_0677_b200/$L timeout 600 python bench.py --config 3 --no-cpu --no-e2e --no-layout --steps 1 --warmup 1 > /tmp/b.json 2>/dev/null
  python -c "
import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); f=d['fp64']; print('$L', f['value'], f['kernel_ms'])"
done
