#!/bin/bash
# K2tcpp with the weight reload barrier (24 B spills instead of 676 B): quick parity, A/B on c4 / c3 / c5.
TAG=r2w
mkdir -p gpurun_out
O=gpurun_out/${TAG}.txt
: > $O
V=paper_2404_19760_b200/variants
LP_LIB_PATH=$V/lib_pp2.so timeout 600 python scripts/sanitize_case.py c4 4096 16 >> $O 2>&1; echo "quick c4 rc=$?" >> $O
for C in c4 c3 c5; do bash scripts/ab_cfg.sh $C paper_2404_19760_b200/liblp_b200.so $V/lib_pp2.so >> $O 2>&1; done
cat $O
