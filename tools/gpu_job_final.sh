#!/bin/bash
# Final validation: smoke, full GPU suite, round artefacts.
set -x
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/smoke.log 2>&1
tail -2 gpurun_out/smoke.log
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_suite.log 2>&1
tail -5 gpurun_out/gpu_suite.log
bash tools/round_artifacts.sh
