# GPU box: persistent lookup grid + RECD_POOL_SHARE in TrainStep
timeout 900 python -m pytest tests/test_gpu_pool.py tests/test_gpu_step.py tests/test_gpu_graph_batches.py -x -q > gpurun_out/pytest_share.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/pytest_share.log
for rep in 1 2 3; do
  bash tools/ab_env.sh "RECD_POOL_CTAS=16" old
  bash tools/ab_env.sh "" new
done
BENCH_ARGS="--config cfg1" bash tools/ab_env.sh "RECD_POOL_CTAS=16" c1old
BENCH_ARGS="--config cfg1" bash tools/ab_env.sh "" c1new
