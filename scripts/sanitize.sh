#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over every kernel family
# (SURVEY section 4, T8), with the persistent grid capped (LP_MAX_CTAS) so each
# group marches several tiles and the scatter-warp hand-offs cycle.
# Logs: gpurun_out/sanitize_<tool>_<case>.log, summary gpurun_out/sanitize_summary.txt
set -u
OUT=${OUT:-gpurun_out}
mkdir -p "$OUT"
CS=/usr/local/cuda/bin/compute-sanitizer
SUM=$OUT/sanitize_summary.txt
: > "$SUM"
# case: cfg rays S   (K2tc K=8/16/32 triplane+voxel, K2tc2, K2tcv, Splatter, g_s Splatter)
CASES_MEM="c1:2048:32 c2:1024:24 c4:1024:24 c5:512:16 c4p:768:16 cu:512:16 c4v:768:16 c1v:1024:16 s1:512:16 s2:512:16 s1g:256:12 s2g:256:12"
CASES_RACE="c1:1024:8 c4:1024:6 c2:512:6 c4p:512:5 c4v:512:5 s2g:256:4 s1:256:6"
run() {   # tool cap case extra
  local tool=$1 cap=$2 c=$3; shift 3
  IFS=: read -r cfg n s <<< "$c"
  local log=$OUT/sanitize_${tool}_${cfg}.log
  local t0=$(date +%s)
  LP_MAX_CTAS=$cap timeout 1500 $CS --tool "$tool" "$@" --print-limit 50 python scripts/sanitize_case.py "$cfg" "$n" "$s" > "$log" 2>&1
  local rc=$?
  local t1=$(date +%s)
  echo "$tool $cfg n=$n S=$s LP_MAX_CTAS=$cap rc=$rc $((t1 - t0))s :: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' "$log" | tail -1)" | tee -a "$SUM"
}
for c in $CASES_MEM; do run memcheck 2 "$c" --leak-check no; done
for c in $CASES_MEM; do run synccheck 2 "$c"; done
for c in $CASES_RACE; do run racecheck 1 "$c" --racecheck-report hazard; done
