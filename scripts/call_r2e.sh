#!/bin/bash
# every-lane drained arrivals: racecheck + parity; K2tc2 producer-kernel A/B variants
mkdir -p gpurun_out
O=gpurun_out/r2e.txt
: > $O
CS=/usr/local/cuda/bin/compute-sanitizer
for c in c4:1024:6 c2:512:6 c4p:512:5 s2g:256:4 c4v:512:5; do
  IFS=: read -r cfg n s <<< "$c"
  LP_MAX_CTAS=1 timeout 900 $CS --tool racecheck --racecheck-report hazard --print-limit 20 python scripts/sanitize_case.py $cfg $n $s > gpurun_out/r2e_race_$cfg.log 2>&1
  echo "racecheck $cfg rc=$? :: $(grep -E 'RACECHECK SUMMARY' gpurun_out/r2e_race_$cfg.log | tail -1)" >> $O
done
timeout 1500 python -m pytest -q -x --timeout 900 tests/test_gpu_parity.py tests/test_gpu_multitile.py tests/test_gpu_splat.py -k "c4 or c2 or c4p or splat_mlp or view" > gpurun_out/r2e_tests.log 2>&1
tail -2 gpurun_out/r2e_tests.log >> $O
for c in c4p; do bash scripts/ab_cfg.sh $c paper_2404_19760_b200/variants/lib_tc2old.so paper_2404_19760_b200/liblp_b200.so paper_2404_19760_b200/variants/lib_u1.so paper_2404_19760_b200/variants/lib_sw2.so paper_2404_19760_b200/variants/lib_nosc.so >> $O 2>&1; done
cat $O
