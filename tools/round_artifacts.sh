#!/bin/bash
# Round-end measurement bundle (run under gpurun from the repo root):
# bench line, reference arm, launch list, ncu --set full of the top kernels,
# parity report.  Outputs in gpurun_out/ (copied to profiles/ by hand).
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -c 400 gpurun_out/bench.json
python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
tail -c 400 gpurun_out/bench_ref.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu --no-fp64 > gpurun_out/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:mls_tc_kernel -s 1 -c 1 -o gpurun_out/mls_tc_full -f \
    python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-layout --no-fp64 > gpurun_out/ncu_mls.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:bh_kernel -s 20 -c 1 -o gpurun_out/bh_full -f \
    python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e --no-fp64 --layout-iters 30 > gpurun_out/ncu_bh.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"^local_kernel" -s 3 -c 1 -o gpurun_out/local_full -f \
    python tools/prof_layout.py 3 > gpurun_out/ncu_local.log 2>&1
MDC_PROF_ROWS=64 ncu --set full --import-source on --clock-control none -k regex:mls_kernel -c 1 -o gpurun_out/mls_f64_full -f \
    python tools/prof_fp64.py > gpurun_out/ncu_f64.log 2>&1
python -m pytest tests/test_gpu_parity_report.py tests/test_gpu_bench_parity.py -q -s -m gpu -p no:cacheprovider > gpurun_out/parity.log 2>&1
ls -la gpurun_out
