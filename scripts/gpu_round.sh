#!/bin/bash
# One GPU session: parity tests, cfg3 bench (+ncu), extra configs. Output -> gpurun_out/
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -25 | tee gpurun_out/gpu_tests.log
for c in ${CONFIGS:-cfg3}; do
  timeout 900 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 ${BENCH_ARGS} > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.log
  echo "bench $c rc=$?"; cat gpurun_out/bench_$c.json; tail -3 gpurun_out/bench_$c.log
done
if [ -n "$NCU_CONFIG" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"psa_|pyramid|importance|assign|antidiag|simcap" \
     --csv --log-file gpurun_out/launches.csv python bench.py --config $NCU_CONFIG --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_bench.log 2>&1
  echo "ncu launches rc=$?"
  for k in ${NCU_KERNELS:-psa_attn_fwd}; do
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 \
       -o gpurun_out/${k}_full -f python bench.py --config $NCU_CONFIG --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_$k.log 2>&1
    echo "ncu $k rc=$?"
  done
fi
