set -x
mkdir -p gpurun_out
./tools/utest_approx
timeout 900 python -m pytest tests/test_gpu_layout.py -q -p no:cacheprovider 2>&1 | tail -3
timeout 300 python bench.py --config 1 --no-cpu --no-e2e --no-fp64 > gpurun_out/bench_c1_r2d.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/bench_c1_r2d.json').read().strip().splitlines()[-1]); print('c1 layout', d['layout']['value'], d['layout']['ms_total'], 'mls', d['value'])"
for L in libmdc.so libmdc_newton1.so; do
  MDC_LIB_PATH=$PWD/paper_1408_0677_b200/$L timeout 300 python bench.py --config 3 --no-cpu --no-e2e --no-fp64 --steps 1 --warmup 1 > gpurun_out/bench_lay_$L.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/bench_lay_$L.json').read().strip().splitlines()[-1]); L=d['layout']; print('$L', L['value'], L['roofline']['phases_ms_one_eager_step']['bh_traversal'], L['roofline']['bh']['frac'])"
done
MDC_LIB_PATH=$PWD/paper_1408_0677_b200/libmdc_newton1.so timeout 900 python -m pytest tests/test_gpu_layout.py tests/test_gpu_seam.py -q -p no:cacheprovider 2>&1 | tail -3
