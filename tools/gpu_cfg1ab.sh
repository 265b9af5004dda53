# cfg1 latency A/B: local (one-CTA) small sorts, 256-row numbering chunks, 32-position scatter / 16-position grad_u tasks
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sort.py tests/test_gpu_step.py tests/test_gpu_bwd.py tests/test_gpu_dedup.py tests/test_gpu_graph_batches.py tests/test_gpu_runs.py tests/test_gpu_pool.py tests/test_gpu_jagged.py -m gpu -x -q > gpurun_out/c1ab_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/c1ab_pytest.log
RECD_LIB=build/variants/librecd_gu16rc32.so timeout 600 python -m pytest tests/test_gpu_step.py tests/test_gpu_bwd.py -m gpu -x -q > gpurun_out/c1ab_pytest_v.log 2>&1; echo pytest gu16rc32 rc=$?; tail -1 gpurun_out/c1ab_pytest_v.log
for rep in 1 2; do BENCH_ARGS="--config cfg1 --steps 300 --warmup 30" bash tools/ab.sh "" cur nolocal nbbig rc32 gu16 gu16rc32; done
bash tools/ab.sh "" cur
