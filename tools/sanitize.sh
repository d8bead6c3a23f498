#!/bin/bash
# compute-sanitizer over every kernel family (tools/san_workload.py) and the
# two-process peer/all-gather layout tests; summaries -> gpurun_out/san_*.log
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 $CS --tool $tool --print-limit 20 python tools/san_workload.py > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' gpurun_out/san_$tool.log | tail -2 | tr '\n' ' ')"
done
timeout 1200 $CS --tool memcheck --target-processes all --print-limit 20 python -m pytest tests/test_gpu_layout_p2p.py -q -x -k "not 1m" > gpurun_out/san_memcheck_p2p.log 2>&1
echo "memcheck p2p rc=$? $(grep -E 'ERROR SUMMARY|passed|failed' gpurun_out/san_memcheck_p2p.log | tail -3 | tr '\n' ' ')"
