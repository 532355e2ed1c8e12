# Full evidence pass on the current build: bash scripts/round_evidence.sh <tag>
# bench (c4, with cpu baseline + e2e), reference arm, launch list, ncu full + traffic for c4 and c4p.
TAG=${1:-r1}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_${TAG}.json 2> gpurun_out/bench_ref_${TAG}.err
for C in c4 c4p; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}_${C}.csv \
      python bench.py --config $C --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/launches_${TAG}_${C}.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:lp_ -s 2 -c 2 -o gpurun_out/prof_${TAG}_${C} -f \
      python scripts/profile_step.py --config $C --rays 524288 --iters 2 > gpurun_out/prof_${TAG}_${C}.log 2>&1
  ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_red.sum -k regex:lp_ \
      python scripts/profile_step.py --config $C --rays 1048576 --iters 2 > gpurun_out/traffic_${TAG}_${C}.txt 2>&1
done
tail -1 gpurun_out/bench_${TAG}.json
