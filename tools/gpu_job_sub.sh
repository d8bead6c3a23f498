#!/bin/bash
for L in libmdc.so libmdc_sub512.so libmdc_sub2048.so libmdc_sub4096.so libmdc_cl8.so; do
  for c in 2 3; do MDC_LIB_PATH=$PWD/paper_1408_0677_b200/$L timeout 300 python tools/prof_layout.py $c 2>&1 | grep graph | sed "s/^/$L c$c /"; done
done
