#!/bin/bash
# Conflict-free paired H-tile stores (LP_GATHER_LANES=1): parity of the variant library, then A/B;
# paired stores in K1tcv/K2tcv (LP_TCV_PAIR=1); the precision guard with the slack-adjusted L2.
TAG=r2s
mkdir -p gpurun_out
O=gpurun_out/${TAG}.txt
: > $O
V=paper_2404_19760_b200/variants
LP_LIB_PATH=$V/lib_lanes1_tcvpair.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multitile.py -m gpu -q --timeout 900 \
    -k "parity_subset or view_dependent or capped_grid or fwd_bwd_host" > gpurun_out/${TAG}_tests_lanes1.log 2>&1
echo "lanes1+tcvpair parity: $(tail -1 gpurun_out/${TAG}_tests_lanes1.log)" >> $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 900 -k "gradient_precision" > gpurun_out/${TAG}_tests_prec.log 2>&1
echo "precision guard: $(tail -1 gpurun_out/${TAG}_tests_prec.log)" >> $O
for C in c4 c3 c4p cu c4pv; do bash scripts/ab_cfg.sh $C paper_2404_19760_b200/liblp_b200.so $V/lib_lanes1.so >> $O 2>&1; done
bash scripts/ab_cfg.sh c4v paper_2404_19760_b200/liblp_b200.so $V/lib_lanes1.so $V/lib_lanes1_tcvpair.so >> $O 2>&1
cat $O
