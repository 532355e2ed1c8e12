#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out/r2o.txt
: > $O
for c in c4:4096:32 c2:2048:32 c5:1024:16; do IFS=: read -r cfg n s <<< "$c"
  timeout 120 python scripts/sanitize_case.py $cfg $n $s > gpurun_out/r2o_quick_$cfg.log 2>&1; echo "quick $cfg rc=$?" >> $O; tail -1 gpurun_out/r2o_quick_$cfg.log >> $O; done
if ! grep -q "rc=124" $O; then
timeout 1200 python -m pytest -q -x --timeout 300 tests/test_gpu_parity.py tests/test_gpu_multitile.py -k "not c4p and not c3p and not cu and not view" > gpurun_out/r2o_tests.log 2>&1
tail -2 gpurun_out/r2o_tests.log >> $O
for c in c4 c3 c2; do bash scripts/ab_cfg.sh $c paper_2404_19760_b200/variants/lib_prev.so paper_2404_19760_b200/liblp_b200.so >> $O 2>&1; done
LP_LIB_PATH=paper_2404_19760_b200/variants/lib_phases.so timeout 300 python scripts/phases.py c4 8388608 >> $O 2>&1
fi
cat $O
