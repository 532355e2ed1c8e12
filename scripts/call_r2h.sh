#!/bin/bash
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:lp_bwd_tc2p -c 1 -o gpurun_out/prof_r2h_c4p -f \
    python scripts/profile_step.py --config c4p --rays 524288 --iters 1 > gpurun_out/prof_r2h_c4p.log 2>&1
python scripts/ncu_summary.py gpurun_out/prof_r2h_c4p.ncu-rep > gpurun_out/prof_r2h_c4p.md 2>&1
ncu -i gpurun_out/prof_r2h_c4p.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_r2h_c4p_sass.csv 2>/dev/null
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2h_c4p.csv \
    python bench.py --config c4p --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/launches_r2h_c4p.log 2>&1
cat gpurun_out/prof_r2h_c4p.md
ls -la gpurun_out/prof_r2h_c4p*
