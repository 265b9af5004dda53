# GPU box: scatter one-task-per-warp default vs old grid-stride cap
timeout 600 python -m pytest tests/test_gpu_bwd.py tests/test_gpu_step.py tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest_sc.log 2>&1
echo "pytest rc=$?"; tail -1 gpurun_out/pytest_sc.log
for rep in 1 2 3; do
  bash tools/ab_env.sh "RECD_SC_CTAS=16" old
  bash tools/ab_env.sh "" new
done
BENCH_ARGS="--config cfg1" bash tools/ab_env.sh "RECD_SC_CTAS=16" c1old
BENCH_ARGS="--config cfg1" bash tools/ab_env.sh "" c1new
