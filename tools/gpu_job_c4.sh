#!/bin/bash
for L in libmdc.so libmdc_radix.so; do MDC_LIB_PATH=$PWD/paper_1408_0677_b200/$L timeout 600 python tools/prof_layout.py 4 2>&1 | grep graph | sed "s/^/$L c4 /"; done
