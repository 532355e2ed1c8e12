#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out/r2k.txt
: > $O
V=paper_2404_19760_b200/variants
bash scripts/ab_cfg.sh c4p paper_2404_19760_b200/liblp_b200.so $V/lib_phc.so $V/lib_anc_all.so $V/lib_anc_24.so $V/lib_anc_3.so >> $O 2>&1
cat $O
