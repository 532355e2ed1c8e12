#!/bin/bash
# Round-2 batch: TMEM-A MMA probe, BASELINE.md section 2 table (every BASELINE config with its
# N-thread and 1-thread oracle rates), the reference arm, compute-sanitizer over every kernel family.
mkdir -p gpurun_out
./scripts/tc_probe3 > gpurun_out/tc_probe3.txt 2>&1; cat gpurun_out/tc_probe3.txt
for c in c1 c2 c3 c5; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --cpu-seconds 10 > gpurun_out/base_$c.json 2> gpurun_out/base_$c.err
  tail -c 600 gpurun_out/base_$c.json
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_c4.json 2> gpurun_out/bench_ref_c4.err
tail -c 400 gpurun_out/bench_ref_c4.json
OUT=gpurun_out bash scripts/sanitize.sh
cat gpurun_out/sanitize_summary.txt
