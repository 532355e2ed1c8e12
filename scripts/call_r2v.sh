#!/bin/bash
# K2tcpp (ping-pong halves over the K2tcp producer design): parity of the variant library, then A/B.
TAG=r2v
mkdir -p gpurun_out
O=gpurun_out/${TAG}.txt
: > $O
V=paper_2404_19760_b200/variants
LP_LIB_PATH=$V/lib_pp.so timeout 600 python scripts/sanitize_case.py c4 4096 16 >> $O 2>&1; echo "quick c4 rc=$?" >> $O
LP_LIB_PATH=$V/lib_pp.so LP_MAX_CTAS=2 timeout 600 python scripts/sanitize_case.py c5 2048 12 >> $O 2>&1; echo "quick c5 capped rc=$?" >> $O
LP_LIB_PATH=$V/lib_pp.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multitile.py -m gpu -q --timeout 900 \
    -k "c4 or c3 or c5 or fwd_bwd_host" > gpurun_out/${TAG}_tests_pp.log 2>&1
echo "pp parity: $(tail -1 gpurun_out/${TAG}_tests_pp.log)" >> $O
for C in c4 c3 c5; do bash scripts/ab_cfg.sh $C paper_2404_19760_b200/liblp_b200.so $V/lib_pp.so >> $O 2>&1; done
cat $O
