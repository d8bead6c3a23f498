#!/bin/bash
# A/B the MLS kernel across candidate libmdc builds (experiments only).
for L in "$@"; do
  MDC_LIB_PATH=$PWD/paper_1408_0677_b200/$L timeout 300 python bench.py --frame 1920x1080 --no-layout --no-cpu --no-e2e --steps 3 --warmup 1 \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$L', round(d['value'],1), round(d['roofline']['kernel_ms'],1), d['clocks']['sm_mhz'])"
done
