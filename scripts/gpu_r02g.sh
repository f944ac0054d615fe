cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -5 | tee gpurun_out/r02g_tests.log
for c in cfg3 cfg4; do
timeout 600 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/r02g_bench_$c.json 2> gpurun_out/r02g_bench_$c.log; echo "rc $c $?"
done
timeout 600 python bench.py --impl reference --config cfg3 --steps 3 --warmup 1 > gpurun_out/r02g_ref_cfg3.json 2> gpurun_out/r02g_ref_cfg3.log; echo "rc ref $?"
