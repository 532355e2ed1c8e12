# usage: bash scripts/ncu_tc.sh <tag> [config] [rays]
set -x
TAG=${1:-r1tc}; CFG=${2:-c4}; RAYS=${3:-524288}
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:lp_ -s 2 -c 2 -o gpurun_out/prof_${TAG} -f     python scripts/profile_step.py --config $CFG --rays $RAYS --iters 2 > gpurun_out/prof_${TAG}.log 2>&1
tail -3 gpurun_out/prof_${TAG}.log
