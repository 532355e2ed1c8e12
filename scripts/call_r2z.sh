#!/bin/bash
# A/B: K2tcp with the compute-role clock anchors (LP_TCP_ANCHOR=1) and with 2 scatter warps.
TAG=r2z
mkdir -p gpurun_out
O=gpurun_out/${TAG}.txt
: > $O
V=paper_2404_19760_b200/variants
for C in c4 c3 c5; do bash scripts/ab_cfg.sh $C paper_2404_19760_b200/liblp_b200.so $V/lib_anchor.so $V/lib_tcpsw2.so >> $O 2>&1; done
bash scripts/ab_cfg.sh c4 paper_2404_19760_b200/liblp_b200.so $V/lib_anchor.so >> $O 2>&1
cat $O
