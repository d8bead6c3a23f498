#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 300 python tools/prof_layout.py 2
timeout 300 python tools/prof_layout.py 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python tools/prof_layout.py 2 > /dev/null 2>&1
python tools/summarize_launches.py gpurun_out/launches_c2.csv | head -25
