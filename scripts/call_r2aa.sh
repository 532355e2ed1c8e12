#!/bin/bash
# A/B of the scatter-warp count: K2tcp (c4, 1 / 2 / 4), K2tc2 (c4p, 2 / 4), K2tcv (c4v, 2 / 4), g_s Splatter (s1g, s2g).
TAG=r2aa
mkdir -p gpurun_out
O=gpurun_out/${TAG}.txt
: > $O
V=paper_2404_19760_b200/variants
M=paper_2404_19760_b200/liblp_b200.so
bash scripts/ab_cfg.sh c4 $M $V/lib_tcpsw2.so $V/lib_tcpsw1.so $M $V/lib_tcpsw2.so >> $O 2>&1
bash scripts/ab_cfg.sh c4p $M $V/lib_tc2sw2.so >> $O 2>&1
bash scripts/ab_cfg.sh cu $M $V/lib_tc2sw2.so >> $O 2>&1
bash scripts/ab_cfg.sh c4v $M $V/lib_tcvsw2.so >> $O 2>&1
for C in s1g s2g; do
  for L in $M $V/lib_gssw2.so; do
    echo "== $C $L" >> $O
    LP_LIB_PATH=$L timeout 600 python bench.py --config $C --steps 3 --warmup 2 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,3), 'M rays/s', {k: round(v,1) for k,v in d['breakdown_ms'].items()})" >> $O 2>&1
  done
done
cat $O
