#!/bin/bash
# K2tc2 with split commits (LP_TC2P_SPLIT=1): parity of the variant, A/B on c4p / cu / c3p.
TAG=r2ag
mkdir -p gpurun_out
O=gpurun_out/${TAG}.txt
: > $O
V=paper_2404_19760_b200/variants
M=paper_2404_19760_b200/liblp_b200.so
LP_LIB_PATH=$V/lib_split.so LP_MAX_CTAS=2 timeout 600 python scripts/sanitize_case.py c4p 2048 12 >> $O 2>&1; echo "quick c4p capped rc=$?" >> $O
LP_LIB_PATH=$V/lib_split.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multitile.py -m gpu -q --timeout 900 \
    -k "c4p or c3p or cu" > gpurun_out/${TAG}_tests.log 2>&1
echo "split parity: $(tail -1 gpurun_out/${TAG}_tests.log)" >> $O
bash scripts/ab_cfg.sh c4p $M $V/lib_split.so $M $V/lib_split.so >> $O 2>&1
bash scripts/ab_cfg.sh cu $M $V/lib_split.so >> $O 2>&1
bash scripts/ab_cfg.sh c3p $M $V/lib_split.so >> $O 2>&1
cat $O
