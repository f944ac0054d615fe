cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -3 > gpurun_out/gpu_tests.log
cat gpurun_out/gpu_tests.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.log
echo "bench rc=$?"
timeout 300 python scripts/probes/bwd_probe.py 2>&1 | grep -v "Warn\|warn_once" > gpurun_out/bwd_probe.log
echo "bwd probe rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:psa_bwd_dkv_tc -s 2 -c 1 \
   -o gpurun_out/psa_bwd_dkv_tc_full -f python scripts/probes/bwd_probe.py > gpurun_out/ncu_bwd_dkv.log 2>&1
echo "ncu bwd_dkv rc=$?"
timeout 600 ncu --section SpeedOfLight --section WarpStateStats --section ComputeWorkloadAnalysis --clock-control none -k regex:psa_bwd_dq_tc -s 2 -c 1 \
   python scripts/probes/bwd_probe.py > gpurun_out/ncu_bwd_dq.log 2>&1
echo "ncu bwd_dq rc=$?"
