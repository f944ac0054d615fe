#!/bin/bash
# Importance-kernel iteration: the tests that pin the importance scores / level maps, cfg3 + cfg4
# bench lines (stage times), and one ncu source-level capture of the antidiagonal xl_stats launch.
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
TAG=${TAG:-xl}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_fullshape.py tests/test_gpu_workunits.py -q -x -p no:cacheprovider 2>&1 | tail -4 | tee gpurun_out/${TAG}_tests.log
for c in cfg3 cfg4; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-yardsticks > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.log
  python -c "import json; d=json.load(open('gpurun_out/${TAG}_bench_$c.json')); print('$c', round(d['ms_per_step'],3), d['stage_ms'])" || tail -5 gpurun_out/${TAG}_bench_$c.log
done
if [ -n "$NCU" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:xl_stats -s 3 -c 1 \
   -o gpurun_out/${TAG}_xl_antidiag -f python bench.py --config cfg4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-yardsticks > gpurun_out/${TAG}_ncu.log 2>&1
echo "ncu rc=$?"
fi
