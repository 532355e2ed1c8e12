# usage: bash scripts/ncu_round.sh <tag> [config] [rays]
set -x
TAG=${1:-r1}; CFG=${2:-c4}; RAYS=${3:-524288}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --config $CFG > gpurun_out/launches_${TAG}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:lp_ -s 2 -c 2 -o gpurun_out/prof_${TAG} -f \
    python scripts/profile_step.py --config $CFG --rays $RAYS --iters 2 > gpurun_out/prof_${TAG}.log 2>&1
ls -la gpurun_out
