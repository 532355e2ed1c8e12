#!/bin/bash
# A/B: K1tc2 forward gather unroll 1 / 2 / 4 (c4p, c3p, cu).
TAG=r2al
mkdir -p gpurun_out
O=gpurun_out/${TAG}.txt
: > $O
V=paper_2404_19760_b200/variants
M=paper_2404_19760_b200/liblp_b200.so
for C in c4p c3p cu; do bash scripts/ab_cfg.sh $C $M $V/lib_f2u1.so $V/lib_f2u4.so >> $O 2>&1; done
bash scripts/ab_cfg.sh c4p $M $V/lib_f2u1.so $V/lib_f2u4.so >> $O 2>&1
cat $O
