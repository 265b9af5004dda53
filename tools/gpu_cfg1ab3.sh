# cfg1 latency A/B 3: fused small inverse CSR (cur vs noinvl), fused expansion through the CSR at cfg1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sort.py tests/test_gpu_step.py tests/test_gpu_bwd.py tests/test_gpu_dedup.py tests/test_gpu_graph_batches.py tests/test_gpu_runs.py tests/test_gpu_pool.py tests/test_gpu_jagged.py tests/test_gpu_stats.py tests/test_gpu_encoder.py -m gpu -x -q > gpurun_out/c1ab3_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/c1ab3_pytest.log
for rep in 1 2; do
  BENCH_ARGS="--config cfg1 --steps 300 --warmup 30" bash tools/ab.sh "" cur noinvl
  BENCH_ARGS="--config cfg1 --steps 300 --warmup 30" bash tools/ab_env.sh "RECD_FUSED_EXPAND=1" fx1
done
bash tools/ab.sh "" cur
