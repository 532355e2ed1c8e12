#!/bin/bash
# A/B: K2tc2 producers' gather without paired stores, and with unroll 1 (after the split commits).
TAG=r2ak
mkdir -p gpurun_out
O=gpurun_out/${TAG}.txt
: > $O
V=paper_2404_19760_b200/variants
M=paper_2404_19760_b200/liblp_b200.so
bash scripts/ab_cfg.sh c4p $M $V/lib_tc2nopair.so $V/lib_tc2u1.so $M $V/lib_tc2nopair.so $V/lib_tc2u1.so >> $O 2>&1
cat $O
