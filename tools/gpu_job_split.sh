for L in libmdc.so libmdc_split2.so; do
  for fr in 1920x1080 3840x2160; do
    MDC_LIB_PATH=$PWD/paper_1408_0677_b200/$L timeout 300 python bench.py --frame $fr --no-layout --no-cpu --no-e2e --no-fp64 --steps 3 --warmup 3 2>/dev/null \
     | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$L $fr', round(d['value'],1), round(d['roofline']['kernel_ms'],1), d['clocks']['sm_mhz'])"
  done
done
MDC_LIB_PATH=$PWD/paper_1408_0677_b200/libmdc_split2.so timeout 900 python -m pytest tests/test_gpu_mls.py tests/test_gpu_bench_parity.py -q -s -p no:cacheprovider -k "not config5" 2>&1 | grep -E "passed|failed|worst|normwise"
