# usage: bash scripts/round_profile.sh <tag>   -- launch list (bench command) + ncu --set full on K1tc/K2tc
set -x
TAG=${1:-r1}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/launches_${TAG}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:lp_ -s 2 -c 2 -o gpurun_out/prof_${TAG} -f \
    python scripts/profile_step.py --config c4 --rays 524288 --iters 2 > gpurun_out/prof_${TAG}.log 2>&1
ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_red.sum -k regex:lp_ \
    python scripts/profile_step.py --config c4 --rays 1048576 --iters 2 > gpurun_out/traffic_${TAG}.txt 2>&1
tail -3 gpurun_out/prof_${TAG}.log
