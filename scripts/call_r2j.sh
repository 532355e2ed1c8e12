#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out/r2j.txt
: > $O
V=paper_2404_19760_b200/variants
bash scripts/ab_cfg.sh c4p paper_2404_19760_b200/liblp_b200.so $V/lib_phases.so $V/lib_phc.so $V/lib_php.so $V/lib_phs.so $V/lib_fence.so >> $O 2>&1
cat $O
