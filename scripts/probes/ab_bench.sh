#!/bin/bash
# A/B of libpsa variants (attention or importance kernels): same bench (cfg3) with PSA_LIB_PATH pointing at each build in
# scripts/probes/ab/, interleaved twice. Prints attention ms, step ms and the median SM clock.
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
for rep in 1 2; do
  for lib in scripts/probes/ab/libpsa_*.so; do
    PSA_LIB_PATH=$lib timeout 300 python bench.py --config ${CFG:-cfg3} --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-yardsticks > /tmp/ab.json 2>/tmp/ab.log
    python -c "import json; d=json.load(open('/tmp/ab.json')); print('$lib', d['stage_ms'], 'step', d['ms_per_step'], 'sm_mhz', d['clocks']['sm_mhz'])" || tail -3 /tmp/ab.log
  done
done
