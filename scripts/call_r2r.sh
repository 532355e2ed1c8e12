#!/bin/bash
# K1tcv2 / K2tcv2 (view-dependent 3-layer nets): TMEM 16x32bx2 probe, a first parity run, the GPU
# tests of the new configs, sanitizers, bench lines.
TAG=r2r
mkdir -p gpurun_out
O=gpurun_out/${TAG}.txt
: > $O
timeout 120 ./scripts/tc_probe4 >> $O 2>&1
echo "== quick parity cuv" >> $O
timeout 600 python scripts/sanitize_case.py cuv 512 16 >> $O 2>&1; echo "rc=$?" >> $O
echo "== quick parity c4pv (capped grid)" >> $O
LP_MAX_CTAS=2 timeout 600 python scripts/sanitize_case.py c4pv 1024 12 >> $O 2>&1; echo "rc=$?" >> $O
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 > gpurun_out/${TAG}_tests.log 2>&1
tail -3 gpurun_out/${TAG}_tests.log >> $O
for tool in memcheck synccheck; do
  LP_MAX_CTAS=2 timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 50 \
      python scripts/sanitize_case.py cuv 512 12 > gpurun_out/${TAG}_sanitize_${tool}_cuv.log 2>&1
  echo "$tool cuv rc=$? :: $(grep -E 'ERROR SUMMARY' gpurun_out/${TAG}_sanitize_${tool}_cuv.log | tail -1)" >> $O
done
LP_MAX_CTAS=1 timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 50 \
    python scripts/sanitize_case.py cuv 256 5 > gpurun_out/${TAG}_sanitize_racecheck_cuv.log 2>&1
echo "racecheck cuv rc=$? :: $(grep -E 'RACECHECK SUMMARY|ERROR SUMMARY' gpurun_out/${TAG}_sanitize_racecheck_cuv.log | tail -1)" >> $O
bash scripts/configs_bench.sh cuv c4pv >> $O 2>&1
echo "== A/B pair barrier for the half exchange (LP_PAIR_XO 0 vs 1)" >> $O
for C in c4 c4p c4v; do bash scripts/ab_cfg.sh $C paper_2404_19760_b200/variants/lib_xo0.so paper_2404_19760_b200/liblp_b200.so >> $O 2>&1; done
cat $O
