#!/bin/bash
# Round evidence: GPU tests, cfg3 bench (CPU baseline + e2e), other configs, ncu launch list and
# full captures of the three heaviest kernels. Everything lands in gpurun_out/.
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu.txt
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -5 > gpurun_out/gpu_tests.log
cat gpurun_out/gpu_tests.log
timeout 900 python bench.py --config cfg3 --steps 20 --warmup 5 > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.log
echo "bench cfg3 rc=$?"
for c in cfg2 cfg4 cfg1; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.log
  echo "bench $c rc=$?"
done
timeout 600 python bench.py --impl reference --config cfg3 --steps 1 --warmup 0 > gpurun_out/bench_ref_cfg3.json 2> gpurun_out/bench_ref_cfg3.log
echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"psa_|pyramid|importance|assign|antidiag|simcap|xl_|gather" \
   --csv --log-file gpurun_out/launches.csv python bench.py --config cfg3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_bench.log 2>&1
echo "ncu launches rc=$?"
for k in psa_attn_pp2 xl_stats assign_levels pyramid_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 \
     -o gpurun_out/${k}_full -f python bench.py --config cfg3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_$k.log 2>&1
  echo "ncu $k rc=$?"
done
timeout 300 python scripts/probes/bwd_probe.py > gpurun_out/bwd_probe.log 2>&1
echo "bwd probe rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:psa_bwd_dkv_tc -s 2 -c 1 \
   -o gpurun_out/psa_bwd_dkv_tc_full -f python scripts/probes/bwd_probe.py > gpurun_out/ncu_bwd_dkv.log 2>&1
echo "ncu bwd_dkv rc=$?"
