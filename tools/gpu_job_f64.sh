#!/bin/bash
for L in libmdc.so libmdc_f64r1.so libmdc_f64r2.so; do
  MDC_LIB_PATH=$PWD/paper_1408_0677_b200/$L timeout 600 python bench.py --config 3 --no-cpu --no-e2e --no-layout --steps 1 --warmup 1 > /tmp/b.json 2>/dev/null
  python -c "
import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); f=d['fp64']; print('$L', f['value'], f['kernel_ms'], f['roofline']['frac'])"
  MDC_LIB_PATH=$PWD/paper_1408_0677_b200/$L timeout 600 python -m pytest tests/test_gpu_bench_parity.py tests/test_gpu_mls.py -q -p no:cacheprovider -k "fp64 or f64 or double" 2>&1 | tail -1
done
