for L in libmdc.so libmdc_lg8.so libmdc_lg16.so; do
  echo "== $L"; MDC_LIB_PATH=$PWD/paper_1408_0677_b200/$L timeout 300 python tools/prof_small.py 2>&1 | grep "us/step" | head -1
done
for L in libmdc.so libmdc_bh10.so libmdc_bh9.so; do
  MDC_LIB_PATH=$PWD/paper_1408_0677_b200/$L timeout 300 python bench.py --config 3 --no-cpu --no-e2e --no-fp64 --steps 1 --warmup 1 > /tmp/b.json 2>/dev/null
  python -c "import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); L=d['layout']; print('$L', L['value'], L['roofline']['phases_ms_one_eager_step']['bh_traversal'])"
done
MDC_LIB_PATH=$PWD/paper_1408_0677_b200/libmdc_lg8.so timeout 600 python -m pytest tests/test_gpu_layout.py -q -p no:cacheprovider -k "small or teacher_forced_every" 2>&1 | tail -1
