#!/bin/bash
# attention-kernel knob sweep at cfg3 (device timing only)
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for v in ${SWEEP:-"PSA_NONE=0"}; do
  env $v timeout 300 python bench.py --config ${CFG:-cfg3} --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sweep.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/sweep.json')); print('$v', d['ms_per_step'], d['stage_ms']['attention'], d['roofline']['achieved'], d['clocks']['sm_mhz'])"
done
