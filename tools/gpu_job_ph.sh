#!/bin/bash
for L in ${LIBS:-libmdc.so}; do for c in ${CFGS:-3}; do
MDC_LIB_PATH=$PWD/paper_1408_0677_b200/$L timeout 600 python bench.py --config $c --no-cpu --no-e2e --no-fp64 --steps 1 --warmup 1 --layout-iters ${ITERS:-100} > /tmp/b.json 2>/dev/null
python -c "
import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); L=d['layout']; print('$L c$c', L['value'], json.dumps(L['roofline']['phases_ms_one_eager_step']))"
done; done
