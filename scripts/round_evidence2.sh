# Evidence pass for the scatter-warp build: bash scripts/round_evidence2.sh <tag>
# bench c4 (cpu baseline + e2e), reference arm, launch lists (c4, c4p), ncu --set full (c4, c4p),
# cache-warm traffic (c4), every other config's bench line.
TAG=${1:-r1f}
mkdir -p gpurun_out
# measured parity errors (printed by the tests) for the record
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -s -k "parity_subset or view_dependent or density_regimes" \
    > gpurun_out/parity_${TAG}.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_${TAG}.json 2> gpurun_out/bench_ref_${TAG}.err
for C in c4 c4p; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}_${C}.csv \
      python bench.py --config $C --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/launches_${TAG}_${C}.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:lp_ -s 2 -c 2 -o gpurun_out/prof_${TAG}_${C} -f \
      python scripts/profile_step.py --config $C --rays 524288 --iters 2 > gpurun_out/prof_${TAG}_${C}.log 2>&1
done
ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_red.sum -k regex:lp_ \
    python scripts/profile_step.py --config c4 --rays 1048576 --iters 2 > gpurun_out/traffic_${TAG}_c4.txt 2>&1
bash scripts/configs_bench.sh c1v c2 c3 c3p c4p c4v c5 cu s1 s2 s1g s2g > gpurun_out/configs_${TAG}.txt 2>&1
tail -1 gpurun_out/bench_${TAG}.json
cat gpurun_out/configs_${TAG}.txt
