#!/bin/bash
# Adopted scatter-warp counts (K2tcp 2, voxel g_s 2): parity of the affected kernels, bench lines;
# A/B of forward knobs (K1tc groups 3, gather unroll 4).
TAG=r2ab
mkdir -p gpurun_out
O=gpurun_out/${TAG}.txt
: > $O
V=paper_2404_19760_b200/variants
M=paper_2404_19760_b200/liblp_b200.so
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multitile.py tests/test_gpu_splat.py -m gpu -q --timeout 900 \
    -k "c4 or c3 or c5 or splat_mlp or fwd_bwd_host" > gpurun_out/${TAG}_tests.log 2>&1
echo "tests: $(tail -1 gpurun_out/${TAG}_tests.log)" >> $O
bash scripts/configs_bench.sh c4 c3 c5 s1g s2g s1gp >> $O 2>&1
bash scripts/ab_cfg.sh c4 $M $V/lib_fg3.so $V/lib_unroll4.so >> $O 2>&1
cat $O
