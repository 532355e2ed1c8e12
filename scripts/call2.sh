#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest -q -rA --timeout 900 tests/test_gpu_parity.py tests/test_gpu_multitile.py tests/test_gpu_splat.py -k "precision or multitile or host or ragged or splat_mlp" > gpurun_out/c2_tests.log 2>&1
tail -5 gpurun_out/c2_tests.log
LP_LIB_PATH=paper_2404_19760_b200/variants/lib_2piece.so timeout 900 python -m pytest -q -rA --timeout 600 tests/test_gpu_parity.py -k "precision" > gpurun_out/c2_2piece.log 2>&1
tail -3 gpurun_out/c2_2piece.log
for c in c4p c4 c4v cu; do LP_LIB_PATH=paper_2404_19760_b200/variants/lib_phases.so timeout 300 python scripts/phases.py $c 1048576; done > gpurun_out/c2_phases.txt 2>&1
cat gpurun_out/c2_phases.txt
