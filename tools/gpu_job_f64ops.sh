#!/bin/bash
mkdir -p gpurun_out
ncu --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,gpu__time_duration.sum -k regex:mls_kernel --csv python tools/prof_fp64.py > gpurun_out/f64ops.csv 2> gpurun_out/f64ops.err
tail -8 gpurun_out/f64ops.csv
