set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_layout_p2p.py tests/test_gpu_layout.py -q -s -p no:cacheprovider > gpurun_out/tests_r2c.log 2>&1; echo tests rc=$?
grep -E "passed|failed|teacher|free-running" gpurun_out/tests_r2c.log | tail -6
for c in 1 2; do timeout 300 python bench.py --config $c --no-cpu --no-e2e > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; echo c$c rc=$?; done
python - <<'PY'
import json
for c in (1, 2):
    d = json.loads(open(f"gpurun_out/bench_c{c}.json").read().strip().splitlines()[-1])
    print(c, "mls", round(d["value"], 1), "layout", d["layout"]["value"], d["layout"]["ms_total"])
PY
bash tools/sanitize.sh
