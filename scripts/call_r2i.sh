#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out/r2i.txt
: > $O
bash scripts/ab_cfg.sh c4p paper_2404_19760_b200/liblp_b200.so paper_2404_19760_b200/variants/lib_phases.so paper_2404_19760_b200/variants/lib_sw2.so paper_2404_19760_b200/liblp_b200.so >> $O 2>&1
bash scripts/ab_cfg.sh c4 paper_2404_19760_b200/liblp_b200.so >> $O 2>&1
cat $O
