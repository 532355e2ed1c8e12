#!/bin/bash
# The g_s Splatter tests after the gs_case() refactor, incl. the capped-grid multi-tile cases.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_splat.py -m gpu -q -s --timeout 900 > gpurun_out/r2ae_tests.log 2>&1
tail -3 gpurun_out/r2ae_tests.log
