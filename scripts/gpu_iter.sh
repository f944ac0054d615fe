#!/bin/bash
# Quick attention iteration on one GPU: parity tests touching the forward kernel, then the cfg3
# (and optional extra) bench lines without the CPU baseline / e2e legs. Output -> gpurun_out/
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
TAG=${TAG:-iter}
timeout 600 python -m pytest ${TESTS:-tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_fullshape.py} -q -x -p no:cacheprovider 2>&1 | tail -6 | tee gpurun_out/${TAG}_tests.log
for c in ${CONFIGS:-cfg3}; do
  timeout 600 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.log
  echo "bench $c rc=$?"; python -c "import json,sys; d=json.load(open('gpurun_out/${TAG}_bench_$c.json')); print('$c', d['ms_per_step'], d['stage_ms'], d['roofline']['achieved'], d['clocks']['sm_mhz'])" || tail -5 gpurun_out/${TAG}_bench_$c.log
done
