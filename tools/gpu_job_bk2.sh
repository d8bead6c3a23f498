#!/bin/bash
set -x
timeout 900 python -m pytest tests/test_gpu_layout.py tests/test_gpu_layout_p2p.py -q -p no:cacheprovider -x 2>&1 | tail -3
for L in libmdc.so libmdc_lin.so; do
  for c in 2 3 4; do MDC_LIB_PATH=$PWD/paper_1408_0677_b200/$L timeout 300 python tools/prof_layout.py $c 2>&1 | grep graph | sed "s/^/$L c$c /"; done
  MDC_LIB_PATH=$PWD/paper_1408_0677_b200/$L timeout 300 python tools/outlier_sort.py 2>&1 | sed "s/^/$L /"
done
