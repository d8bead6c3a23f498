#!/bin/bash
mkdir -p gpurun_out
for L in libmdc.so libmdc_lin.so; do
MDC_LIB_PATH=$PWD/paper_1408_0677_b200/$L timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"bucket|Scan" -c 30 --csv python tools/prof_layout.py 4 2>/dev/null | grep gpu__time | awk -F'","' '{print $5, $NF}' | sort | awk '{k=$0; sub(/ [0-9.,"]+$/,"",k); v=$NF; gsub(/[",]/,"",v); s[k]+=v; n[k]++} END {for (k in s) print "'$L'", k, n[k], s[k]/n[k]}'
done
