#!/bin/bash
# A/B the layout step phases across candidate libmdc builds (experiments only).
for C in 2 3; do for L in "$@"; do
  MDC_LIB_PATH=$PWD/paper_1408_0677_b200/$L timeout 300 python bench.py --config $C --frame 256x128 --no-cpu --no-e2e --steps 1 --warmup 1 \
    | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); L=d['layout']; print('cfg$C', '$L', round(L['value']/1e6,2), L['orientation_flips'], {k: round(v*1000) for k,v in L['roofline']['phases_ms_one_eager_step'].items()})"
done; done
