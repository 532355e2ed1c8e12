#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out/r2n.txt
: > $O
timeout 120 python scripts/sanitize_case.py c4p 4096 32 > gpurun_out/r2n_quick.log 2>&1
echo "quick c4p rc=$?" >> $O; tail -2 gpurun_out/r2n_quick.log >> $O
if grep -q "rc=0" $O; then
timeout 900 python -m pytest -q -x --timeout 300 tests/test_gpu_parity.py tests/test_gpu_multitile.py -k "c4p or c3p or cu or autograd_render or ragged" > gpurun_out/r2n_tests.log 2>&1
tail -2 gpurun_out/r2n_tests.log >> $O
bash scripts/ab_cfg.sh c4p paper_2404_19760_b200/variants/lib_prev.so paper_2404_19760_b200/liblp_b200.so >> $O 2>&1
bash scripts/ab_cfg.sh cu paper_2404_19760_b200/variants/lib_prev.so paper_2404_19760_b200/liblp_b200.so >> $O 2>&1
fi
cat $O
