#!/bin/bash
# GPU parity tests, then the benchmark (+ optional ncu passes via NCU=1)
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -15 | tee gpurun_out/gpu_tests.log
NCU=${NCU:-0} bash scripts/gpu_bench.sh
