#!/bin/bash
# K1tcv2 with column groups (CG = 2, G = 2 / 1 groups): parity of the vd 3-layer configs, A/B.
TAG=r2u
mkdir -p gpurun_out
O=gpurun_out/${TAG}.txt
: > $O
V=paper_2404_19760_b200/variants
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -k "cuv or c4pv" > gpurun_out/${TAG}_tests.log 2>&1
echo "cuv/c4pv tests (fwd CG=2): $(tail -1 gpurun_out/${TAG}_tests.log)" >> $O
for C in cuv c4pv; do bash scripts/ab_cfg.sh $C $V/lib_fcg1.so paper_2404_19760_b200/liblp_b200.so $V/lib_fg1.so >> $O 2>&1; done
cat $O
