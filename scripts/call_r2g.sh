#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out/r2g.txt
: > $O
timeout 1500 python -m pytest -q -x --timeout 900 tests/test_gpu_parity.py tests/test_gpu_multitile.py -k "c4p or c3p or cu or autograd_render or ragged" > gpurun_out/r2g_tests.log 2>&1
tail -2 gpurun_out/r2g_tests.log >> $O
bash scripts/ab_cfg.sh c4p paper_2404_19760_b200/liblp_b200.so paper_2404_19760_b200/variants/lib_nosc.so >> $O 2>&1
for n in 1048576 8388608; do LP_LIB_PATH=paper_2404_19760_b200/variants/lib_phases.so timeout 300 python scripts/phases.py c4p $n >> $O 2>&1; done
cat $O
