#!/bin/bash
# bench + ncu launch list + one full ncu capture of the attention kernel
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt; lscpu | head -20 >> gpurun_out/nproc.txt
timeout 900 python bench.py --steps ${STEPS:-5} --warmup 3 ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.log
echo "bench rc=$?"; cat gpurun_out/bench.json
if [ "${NCU:-1}" = "1" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"psa_|pyramid|importance|assign" \
   --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS} > gpurun_out/ncu_launch_bench.log 2>&1
echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:psa_attn_fwd -s 3 -c 1 \
   -o gpurun_out/attn_full -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS} > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"
timeout 600 ncu --set full --clock-control none -k regex:importance_stats -s 3 -c 1 \
   -o gpurun_out/imp_full -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS} > gpurun_out/ncu_imp.log 2>&1
echo "ncu imp rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:assign_levels -s 3 -c 1 \
   -o gpurun_out/assign_full -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS} > gpurun_out/ncu_assign.log 2>&1
echo "ncu assign rc=$?"
fi
tail -5 gpurun_out/bench.log
