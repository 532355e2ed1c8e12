#!/bin/bash
# N1 (uniform-cell scatter merge) and N2 (L2 persisting window) A/B, red_bench ceilings
mkdir -p gpurun_out
O=gpurun_out/c3_ab.txt
: > $O
./scripts/red_bench seq >> $O 2>&1
for w in 16 256 0; do ./scripts/red_bench gather $w >> $O 2>&1; done
./scripts/red_bench >> $O 2>&1
for c in c3 c2 c4 c5; do bash scripts/ab_cfg.sh $c paper_2404_19760_b200/liblp_b200.so paper_2404_19760_b200/variants/lib_uniform.so >> $O 2>&1; done
for c in c2 c4 c5; do
  for h in 0.5 1.0; do
    echo "== $c l2_persist $h" >> $O
    timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --l2-persist $h 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,3), 'M rays/s', {k: round(v,1) for k,v in d['breakdown_ms'].items()})" >> $O 2>&1
  done
done
cat $O
