#!/bin/bash
# Round-2 measurement batch: K2tc2/K2tc phase timers, N1 (uniform-cell merge) and N2 (L2
# persisting window) A/B, red_bench gather/seq ceilings, ray-order sensitivity.
mkdir -p gpurun_out
O=gpurun_out/r2b.txt
: > $O
for c in c4p c4 c4v cu; do LP_LIB_PATH=paper_2404_19760_b200/variants/lib_phases.so timeout 300 python scripts/phases.py $c 1048576 >> $O 2>&1; done
echo "== red_bench seq" >> $O; ./scripts/red_bench seq >> $O 2>&1
for w in 16 256 4096 0; do echo "== red_bench gather $w" >> $O; ./scripts/red_bench gather $w >> $O 2>&1; done
echo "== red_bench (random lines)" >> $O; ./scripts/red_bench >> $O 2>&1
for c in c3 c2 c4 c5; do bash scripts/ab_cfg.sh $c paper_2404_19760_b200/liblp_b200.so paper_2404_19760_b200/variants/lib_uniform.so >> $O 2>&1; done
for c in c2 c5 c4; do
  for h in 0.0 0.5 1.0; do
    echo "== $c l2_persist $h" >> $O
    timeout 900 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --l2-persist $h 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,3), 'M rays/s', {k: round(v,1) for k,v in d['breakdown_ms'].items()})" >> $O 2>&1
  done
done
for c in c4 c4p c3; do
  for r in tiled raster shuffled; do
    echo "== $c ray-order $r" >> $O
    timeout 900 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --ray-order $r 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,3), 'M rays/s', {k: round(v,1) for k,v in d['breakdown_ms'].items()}, 'frac', round(d['roofline']['frac'],3))" >> $O 2>&1
  done
done
cat $O
