#!/bin/bash
# The paper's 3-layer g_s Splatter (lp_splat_mlp2_kernels.cuh): parity of every g_s case, bench lines.
TAG=r2x
mkdir -p gpurun_out
O=gpurun_out/${TAG}.txt
: > $O
timeout 1500 python -m pytest tests/test_gpu_splat.py -m gpu -q -s --timeout 900 -k "splat_mlp" > gpurun_out/${TAG}_tests.log 2>&1
echo "g_s tests: $(tail -1 gpurun_out/${TAG}_tests.log)" >> $O
grep "^{" gpurun_out/${TAG}_tests.log | cut -c1-400 >> $O
bash scripts/configs_bench.sh s1gp s2gp s1g s2g >> $O 2>&1
cat $O
