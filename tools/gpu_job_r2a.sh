set -x
mkdir -p gpurun_out
python tools/make_bench_positions.py > gpurun_out/mkpos.log 2>&1; tail -3 gpurun_out/mkpos.log
cp bench_data/*.npz gpurun_out/ 2>/dev/null
timeout 1500 python -m pytest tests -m gpu -q -x -s -p no:cacheprovider > gpurun_out/tests_r2a.log 2>&1; echo tests rc=$?
tail -5 gpurun_out/tests_r2a.log
timeout 400 python bench.py > gpurun_out/bench_r2a.json 2> gpurun_out/bench_r2a.err; echo bench rc=$?
tail -c 1500 gpurun_out/bench_r2a.json
ncu --metrics gpu__time_duration.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum --clock-control none -k regex:mls_kernel --csv python tools/prof_fp64.py > gpurun_out/ncu_fp64_ops.csv 2>&1
ncu --set full --import-source on --clock-control none -k regex:mls_kernel -c 1 -o gpurun_out/mls_fp64_full -f python tools/prof_fp64.py > gpurun_out/ncu_fp64.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"local_kernel|build_levels|build_subtree" -s 30 -c 3 -o gpurun_out/layout_local_full -f python tools/prof_layout.py 3 > gpurun_out/ncu_local.log 2>&1
ls gpurun_out
