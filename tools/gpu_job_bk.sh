#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_layout.py tests/test_gpu_layout_p2p.py -q -p no:cacheprovider -x 2>&1 | tail -3
for L in ${LIBS:-libmdc.so libmdc_nof32.so}; do
  for c in ${CFGS:-2 3}; do MDC_LIB_PATH=$PWD/paper_1408_0677_b200/$L timeout 300 python tools/prof_layout.py $c 2>&1 | grep graph | sed "s/^/$L c$c /"; done
done
for L in ${LIBS:-libmdc.so libmdc_nof32.so}; do
  for c in ${CFGS:-2 3}; do MDC_LIB_PATH=$PWD/paper_1408_0677_b200/$L timeout 300 python tools/prof_layout.py $c 2>&1 | grep graph | sed "s/^/$L c$c /"; done
done
