#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out/r2m.txt
: > $O
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 1200 > gpurun_out/r2m_tests.log 2>&1
tail -2 gpurun_out/r2m_tests.log >> $O
bash scripts/configs_bench.sh c4p cu c3p >> $O 2>&1
LP_LIB_PATH=paper_2404_19760_b200/variants/lib_phases.so timeout 300 python scripts/phases.py c4p 8388608 >> $O 2>&1
cat $O
