#!/bin/bash
# K2tcv2 with split commits (LP_TCV2_SPLIT=1): parity of the variant, A/B on cuv / c4pv.
TAG=r2ai
mkdir -p gpurun_out
O=gpurun_out/${TAG}.txt
: > $O
V=paper_2404_19760_b200/variants
M=paper_2404_19760_b200/liblp_b200.so
LP_LIB_PATH=$V/lib_v2split.so timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -k "cuv or c4pv" > gpurun_out/${TAG}_tests.log 2>&1
echo "v2split parity: $(tail -1 gpurun_out/${TAG}_tests.log)" >> $O
bash scripts/ab_cfg.sh cuv $M $V/lib_v2split.so $M $V/lib_v2split.so >> $O 2>&1
bash scripts/ab_cfg.sh c4pv $M $V/lib_v2split.so >> $O 2>&1
cat $O
