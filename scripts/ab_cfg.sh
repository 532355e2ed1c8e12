# A/B timing of library variants on one config: bash scripts/ab_cfg.sh CONFIG lib1.so lib2.so ...
C=$1; shift
for L in "$@"; do
  echo "== $C $L"
  LP_LIB_PATH=$L timeout 600 python bench.py --config $C --steps 3 --warmup 2 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,3), 'M rays/s', {k: round(v,1) for k,v in d['breakdown_ms'].items()})"
done
