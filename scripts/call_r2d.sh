#!/bin/bash
# K2tc2 producer-warp build: parity of the 3-layer family, then A/B against the single-role kernel
mkdir -p gpurun_out
O=gpurun_out/r2d.txt
: > $O
timeout 1500 python -m pytest -q -x --timeout 900 tests/test_gpu_parity.py tests/test_gpu_multitile.py -k "c4p or c3p or cu or autograd_render or ragged" > gpurun_out/r2d_tests.log 2>&1
tail -3 gpurun_out/r2d_tests.log >> $O
for c in c4p cu c3p; do bash scripts/ab_cfg.sh $c paper_2404_19760_b200/variants/lib_tc2old.so paper_2404_19760_b200/liblp_b200.so >> $O 2>&1; done
for c in c4p cu; do LP_LIB_PATH=paper_2404_19760_b200/variants/lib_phases.so timeout 300 python scripts/phases.py $c 1048576 >> $O 2>&1; done
cat $O
