# ncu evidence for the NEXT-row kernels: bash scripts/evidence_next.sh <tag>
TAG=${1:-r1e}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/tests_${TAG}.log 2>&1; tail -2 gpurun_out/tests_${TAG}.log
for C in c4v s1 s2; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}_${C}.csv \
      python bench.py --config $C --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/launches_${TAG}_${C}.log 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:lp_ -s 2 -c 2 -o gpurun_out/prof_${TAG}_c4v -f \
    python scripts/profile_step.py --config c4v --rays 524288 --iters 2 > gpurun_out/prof_${TAG}_c4v.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:lp_splat -s 3 -c 3 -o gpurun_out/prof_${TAG}_s1 -f \
    python bench.py --config s1 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/prof_${TAG}_s1.log 2>&1
ls gpurun_out | grep $TAG
