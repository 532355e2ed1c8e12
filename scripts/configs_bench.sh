# Bench every config at full size (1 GPU, no cpu baseline / e2e): bash scripts/configs_bench.sh c2 c3 ...
mkdir -p gpurun_out
for c in "$@"; do
  echo "== $c"
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  tail -1 gpurun_out/bench_$c.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,3), 'M rays/s', {k: round(v,1) for k,v in d['breakdown_ms'].items()}, 'frac', round(d['roofline']['frac'],3))" || tail -3 gpurun_out/bench_$c.err
done
