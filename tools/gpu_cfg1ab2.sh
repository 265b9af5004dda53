# cfg1 latency A/B 2: 64-row row-scan blocks (cur vs rs256), 1K-value copy/occurrence blocks (cur vs notiny)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sort.py tests/test_gpu_step.py tests/test_gpu_bwd.py tests/test_gpu_dedup.py tests/test_gpu_graph_batches.py tests/test_gpu_runs.py tests/test_gpu_pool.py tests/test_gpu_jagged.py tests/test_gpu_stats.py tests/test_gpu_partial.py tests/test_gpu_transforms.py -m gpu -x -q > gpurun_out/c1ab2_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/c1ab2_pytest.log
for rep in 1 2; do BENCH_ARGS="--config cfg1 --steps 300 --warmup 30" bash tools/ab.sh "" cur rs256 notiny; done
bash tools/ab.sh "" cur
