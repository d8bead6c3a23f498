set -x
mkdir -p gpurun_out
python tools/make_bench_positions.py > gpurun_out/mkpos.log 2>&1; tail -3 gpurun_out/mkpos.log
cp bench_data/*.npz gpurun_out/ 2>/dev/null
timeout 1800 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/tests_r2b.log 2>&1; echo tests rc=$?
grep -E "passed|failed" gpurun_out/tests_r2b.log | tail -3
timeout 500 python bench.py > gpurun_out/bench_r2b.json 2> gpurun_out/bench_r2b.err; echo bench rc=$?
tail -c 600 gpurun_out/bench_r2b.json
for L in libmdc.so libmdc_nowide.so; do echo "== $L"; MDC_LIB_PATH=$PWD/paper_1408_0677_b200/$L timeout 300 python tools/dsweep.py 2>&1 | grep '"d": \(64\|128\|256\)'; done
ncu --set full --import-source on --clock-control none -k regex:"local_kernel|build_levels|build_subtree" -s 30 -c 3 -o gpurun_out/layout_local_full -f python tools/prof_layout.py 3 > gpurun_out/ncu_local.log 2>&1
ls gpurun_out
