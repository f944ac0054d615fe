timeout 300 python scripts/probes/bwd_probe.py 2>&1 | tail -12
timeout 900 ncu --set full --clock-control none --import-source on -k regex:psa_bwd_dkv_tc -s 2 -c 1 \
   -o gpurun_out/psa_bwd_dkv_tc_full -f python scripts/probes/bwd_probe.py > gpurun_out/ncu_bwd_dkv.log 2>&1
echo "ncu rc=$?"
