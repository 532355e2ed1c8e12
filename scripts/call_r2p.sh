#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out/r2p.txt
: > $O
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 1200 > gpurun_out/r2p_tests.log 2>&1
tail -2 gpurun_out/r2p_tests.log >> $O
bash scripts/ab_cfg.sh c5 paper_2404_19760_b200/variants/lib_prev.so paper_2404_19760_b200/liblp_b200.so >> $O 2>&1
bash scripts/ab_cfg.sh c2 paper_2404_19760_b200/liblp_b200.so >> $O 2>&1
ncu --set full --clock-control none --import-source on -k regex:lp_bwd_tcp -c 1 -o gpurun_out/prof_r2p_c4 -f \
    python scripts/profile_step.py --config c4 --rays 524288 --iters 1 > gpurun_out/prof_r2p_c4.log 2>&1
python scripts/ncu_summary.py gpurun_out/prof_r2p_c4.ncu-rep > gpurun_out/prof_r2p_c4.md 2>&1
ncu -i gpurun_out/prof_r2p_c4.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_r2p_c4_sass.csv 2>/dev/null
cat $O
