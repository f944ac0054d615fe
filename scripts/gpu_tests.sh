cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_parity.py -v -rA -p no:cacheprovider 2>&1 | tee gpurun_out/gpu_tests1.log | tail -120
