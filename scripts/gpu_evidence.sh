#!/bin/bash
# Round evidence on one B200: every GPU test, bench lines (cfg3 full with e2e + CPU baseline +
# parity + yardsticks; cfg1/2/4; cfg5 sweep; reference arm; a 2-rank run), the ncu launch list of
# a cfg3 step and full captures of the heaviest kernels (cfg3; cfg4's antidiagonal xl_stats),
# and the backward probe. Everything lands in gpurun_out/ (summarised by scripts/ncu_summarize.py).
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
T=${TAG:-r02}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/${T}_gpu.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -5 > gpurun_out/${T}_gpu_tests.log
cat gpurun_out/${T}_gpu_tests.log
timeout 900 python bench.py --config cfg3 --steps 20 --warmup 5 > gpurun_out/${T}_bench_cfg3.json 2> gpurun_out/${T}_bench_cfg3.log
echo "bench cfg3 rc=$?"
for c in cfg2 cfg4 cfg1; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/${T}_bench_$c.json 2> gpurun_out/${T}_bench_$c.log
  echo "bench $c rc=$?"
done
timeout 600 python bench.py --config cfg5 --steps 10 --warmup 3 > gpurun_out/${T}_bench_cfg5.json 2> gpurun_out/${T}_bench_cfg5.log
echo "bench cfg5 rc=$?"
timeout 600 python bench.py --impl reference --config cfg3 --steps 3 --warmup 1 > gpurun_out/${T}_bench_ref_cfg3.json 2> gpurun_out/${T}_bench_ref_cfg3.log
echo "ref rc=$?"
timeout 600 python bench.py --gpus 2 --config cfg2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_bench_cfg2_gpus2.json 2> gpurun_out/${T}_bench_cfg2_gpus2.log
echo "gpus2 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
   -k regex:"psa_|pyramid|importance|assign|antidiag|simcap|xl_|gather" --csv --log-file gpurun_out/launches.csv \
   python bench.py --config cfg3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-yardsticks > gpurun_out/${T}_ncu_launch.log 2>&1
echo "ncu launches rc=$?"
for k in psa_attn_pp2 xl_stats assign_levels pyramid_kernel importance_finalize; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 \
     -o gpurun_out/${k}_full -f python bench.py --config cfg3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-yardsticks > gpurun_out/${T}_ncu_$k.log 2>&1
  echo "ncu $k rc=$?"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:xl_stats -s 3 -c 1 \
   -o gpurun_out/xl_stats_antidiag_full -f python bench.py --config cfg4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-yardsticks > gpurun_out/${T}_ncu_xl_antidiag.log 2>&1
echo "ncu xl antidiag rc=$?"
timeout 300 python scripts/probes/bwd_probe.py > gpurun_out/${T}_bwd_probe.log 2>&1
echo "bwd probe rc=$?"
