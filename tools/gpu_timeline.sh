# GPU box: backward stages split -- tests, stream timeline, bench A/B
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_graph_batches.py tests/test_gpu_bwd.py tests/test_gpu_fullsize.py tests/test_gpu_runs.py -x -q > gpurun_out/pytest_stages.log 2>&1
echo "pytest rc=$?"; tail -1 gpurun_out/pytest_stages.log
timeout 300 python tools/timeline.py --steps 10 > gpurun_out/tl_a.txt 2>&1; echo a rc=$?; tail -8 gpurun_out/tl_a.txt
RECD_POOL_CTAS=3 timeout 300 python tools/timeline.py --steps 10 > gpurun_out/tl_b.txt 2>&1; echo b rc=$?; tail -8 gpurun_out/tl_b.txt
for rep in 1 2; do
  bash tools/ab_env.sh "" new
  bash tools/ab_env.sh "RECD_POOL_CTAS=3" pc3
done
