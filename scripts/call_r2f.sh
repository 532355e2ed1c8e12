#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out/r2f.txt
: > $O
timeout 1500 python -m pytest -q -x --timeout 900 tests/test_gpu_parity.py tests/test_gpu_multitile.py -k "c4p or c3p or cu or autograd_render or ragged" > gpurun_out/r2f_tests.log 2>&1
tail -2 gpurun_out/r2f_tests.log >> $O
LP_MAX_CTAS=1 timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 python scripts/sanitize_case.py c4p 512 5 > gpurun_out/r2f_race_c4p.log 2>&1
echo "racecheck c4p :: $(grep -E 'RACECHECK SUMMARY' gpurun_out/r2f_race_c4p.log | tail -1)" >> $O
LP_MAX_CTAS=2 timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool synccheck python scripts/sanitize_case.py c4p 768 16 > gpurun_out/r2f_sync_c4p.log 2>&1
echo "synccheck c4p :: $(grep -E 'ERROR SUMMARY' gpurun_out/r2f_sync_c4p.log | tail -1)" >> $O
for c in c4p cu; do bash scripts/ab_cfg.sh $c paper_2404_19760_b200/variants/lib_tc2old.so paper_2404_19760_b200/liblp_b200.so paper_2404_19760_b200/variants/lib_nosc.so >> $O 2>&1; done
for c in c4p cu; do LP_LIB_PATH=paper_2404_19760_b200/variants/lib_phases.so timeout 300 python scripts/phases.py $c 1048576 >> $O 2>&1; done
cat $O
