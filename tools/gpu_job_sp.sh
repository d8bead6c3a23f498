#!/bin/bash
for c in 2 3; do MDC_LIB_PATH=$PWD/paper_1408_0677_b200/libmdc_sprof.so timeout 300 python tools/prof_layout.py $c 2>&1 | sort | uniq -c | sort -rn | head -4; done
