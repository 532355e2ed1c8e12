#!/bin/bash
# Round-2 evidence of the final build: GPU tests, smoke, c4 bench + reference arm, c4 launch list,
# ncu --set full of c4 (K1tc, K2tcp), cuv (K1tcv2, K2tcv2) and s2gp (3-layer g_s Splatter), cache-warm
# traffic, every config's bench line.
TAG=r2aj
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 > gpurun_out/${TAG}_tests.log 2>&1
tail -2 gpurun_out/${TAG}_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; tail -1 gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench_c4.json 2> gpurun_out/${TAG}_bench_c4.err
tail -1 gpurun_out/${TAG}_bench_c4.json | cut -c1-400
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_ref_c4.json 2> gpurun_out/${TAG}_bench_ref_c4.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_c4.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_launches_c4.log 2>&1
for C in c4:524288 cuv:262144; do
  IFS=: read -r cfg n <<< "$C"
  ncu --set full --clock-control none --import-source on -k regex:lp_ -s 2 -c 2 -o gpurun_out/${TAG}_prof_${cfg} -f \
      python scripts/profile_step.py --config $cfg --rays $n --iters 2 > gpurun_out/${TAG}_prof_${cfg}.log 2>&1
  python scripts/ncu_summary.py gpurun_out/${TAG}_prof_${cfg}.ncu-rep > gpurun_out/${TAG}_ncu_summary_${cfg}.md 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:lp_splat_mlp2 -c 2 -o gpurun_out/${TAG}_prof_s2gp -f \
    python bench.py --config s2gp --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_prof_s2gp.log 2>&1
python scripts/ncu_summary.py gpurun_out/${TAG}_prof_s2gp.ncu-rep > gpurun_out/${TAG}_ncu_summary_s2gp.md 2>&1
ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_red.sum -k regex:lp_ \
    python scripts/profile_step.py --config c4 --rays 1048576 --iters 2 > gpurun_out/${TAG}_traffic_c4_1M.txt 2>&1
bash scripts/configs_bench.sh c1v c2 c3 c3p c4p c4v c5 cu cuv c4pv s1 s2 s1g s2g s1gp s2gp > gpurun_out/${TAG}_configs.txt 2>&1
cat gpurun_out/${TAG}_configs.txt
