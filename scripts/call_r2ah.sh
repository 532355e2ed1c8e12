#!/bin/bash
# K2tcp with split commits (LP_TCP_SPLIT=1): quick parity, A/B on c4 / c3 / c5.
TAG=r2ah
mkdir -p gpurun_out
O=gpurun_out/${TAG}.txt
: > $O
V=paper_2404_19760_b200/variants
M=paper_2404_19760_b200/liblp_b200.so
LP_LIB_PATH=$V/lib_tcpsplit.so LP_MAX_CTAS=2 timeout 600 python scripts/sanitize_case.py c4 4096 12 >> $O 2>&1; echo "quick c4 capped rc=$?" >> $O
bash scripts/ab_cfg.sh c4 $M $V/lib_tcpsplit.so $M $V/lib_tcpsplit.so >> $O 2>&1
bash scripts/ab_cfg.sh c3 $M $V/lib_tcpsplit.so >> $O 2>&1
bash scripts/ab_cfg.sh c5 $M $V/lib_tcpsplit.so >> $O 2>&1
cat $O
