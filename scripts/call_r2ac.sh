#!/bin/bash
# A/B of the cooperative gather's unroll (2 / 4 / 8) over the kernel families that use the default.
TAG=r2ac
mkdir -p gpurun_out
O=gpurun_out/${TAG}.txt
: > $O
V=paper_2404_19760_b200/variants
M=paper_2404_19760_b200/liblp_b200.so
for C in c4 c3 c5 c2 c4p cuv; do bash scripts/ab_cfg.sh $C $M $V/lib_unroll4.so $V/lib_unroll8.so >> $O 2>&1; done
for C in s1g s2g s2gp; do
  for L in $M $V/lib_unroll4.so $V/lib_unroll8.so; do
    echo "== $C $L" >> $O
    LP_LIB_PATH=$L timeout 600 python bench.py --config $C --steps 3 --warmup 2 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,3), 'M rays/s', {k: round(v,1) for k,v in d['breakdown_ms'].items()})" >> $O 2>&1
  done
done
cat $O
