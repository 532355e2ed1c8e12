#!/bin/bash
# HEAD sanity: smoke and the K1tc2 / K2tc2 parity cases after the last knob edits.
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2am_smoke.log 2>&1; tail -1 gpurun_out/r2am_smoke.log | cut -c1-120
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multitile.py -m gpu -q --timeout 900 -k "c4p or c3p or cu" > gpurun_out/r2am_tests.log 2>&1
tail -1 gpurun_out/r2am_tests.log
