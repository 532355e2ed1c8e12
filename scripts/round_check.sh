#!/bin/bash
# GPU round check: smoke, the -m gpu suite, a short bench (logs under gpurun_out/)
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
timeout ${TEST_TIMEOUT:-2400} python -m pytest tests -m gpu -q -rA --timeout 1200 ${PYTEST_ARGS:-} > gpurun_out/tests_gpu.log 2>&1
tail -40 gpurun_out/tests_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -c 3000 gpurun_out/bench.json
