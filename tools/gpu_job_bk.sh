#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_layout.py -q -p no:cacheprovider -x 2>&1 | tail -3
for L in libmdc.so libmdc_nosplit.so libmdc_minb8.so; do
  for c in ${CFGS:-2 3}; do MDC_LIB_PATH=$PWD/paper_1408_0677_b200/$L timeout 300 python tools/prof_layout.py $c 2>&1 | grep -v "^step eager" | sed "s/^/$L c$c /"; done
done
