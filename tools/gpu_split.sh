# inverse CSR and occurrence sort on two streams after RECD_BWD_SETUP (default) vs in series (RECD_SPLIT_PREP=0)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/split_pytest.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/split_pytest.log
RECD_SPLIT_PREP=0 timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_graph_batches.py -m gpu -x -q 2>&1 | tail -1
for rep in 1 2 3; do
  BENCH_ARGS="--config cfg1 --steps 300 --warmup 30" bash tools/ab_env.sh "RECD_SPLIT_PREP=1" c1split
  BENCH_ARGS="--config cfg1 --steps 300 --warmup 30" bash tools/ab_env.sh "RECD_SPLIT_PREP=0" c1serial
done
for rep in 1 2 3; do
  bash tools/ab_env.sh "RECD_SPLIT_PREP=1" c2split
  bash tools/ab_env.sh "RECD_SPLIT_PREP=0" c2serial
done
