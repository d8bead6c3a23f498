#!/bin/bash
mkdir -p gpurun_out
MDC_PROF_ROWS=64 ncu --set full --import-source on --clock-control none -k regex:mls_kernel -c 1 -o gpurun_out/mls_f64_full -f python tools/prof_fp64.py > gpurun_out/ncu_f64.log 2>&1
tail -3 gpurun_out/ncu_f64.log
