#!/bin/bash
# K2tcv2 with two column groups (4 threads per ray, 8 compute warps): parity, then A/B against CG = 1.
TAG=r2t
mkdir -p gpurun_out
O=gpurun_out/${TAG}.txt
: > $O
V=paper_2404_19760_b200/variants
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -k "cuv or c4pv" > gpurun_out/${TAG}_tests.log 2>&1
echo "cuv/c4pv tests (CG=2): $(tail -1 gpurun_out/${TAG}_tests.log)" >> $O
for C in cuv c4pv; do bash scripts/ab_cfg.sh $C $V/lib_cg1.so paper_2404_19760_b200/liblp_b200.so >> $O 2>&1; done
cat $O
