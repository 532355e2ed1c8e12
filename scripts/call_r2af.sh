#!/bin/bash
# A/B: K2tc2 producer gather unroll 4 (c4p, cu); K2tcv2 with one scatter warp (cuv).
TAG=r2af
mkdir -p gpurun_out
O=gpurun_out/${TAG}.txt
: > $O
V=paper_2404_19760_b200/variants
M=paper_2404_19760_b200/liblp_b200.so
bash scripts/ab_cfg.sh c4p $M $V/lib_tc2u4.so $M $V/lib_tc2u4.so >> $O 2>&1
bash scripts/ab_cfg.sh cu $M $V/lib_tc2u4.so >> $O 2>&1
bash scripts/ab_cfg.sh cuv $M $V/lib_v2sw1.so >> $O 2>&1
cat $O
