# PDL launch helper change: GPU suite with PDL forced on, then default; cfg1 bench
mkdir -p gpurun_out
RECD_PDL=1 timeout 900 python -m pytest tests/test_gpu_sort.py tests/test_gpu_dedup.py tests/test_gpu_pool.py tests/test_gpu_step.py tests/test_gpu_bwd.py tests/test_gpu_graph_batches.py -m gpu -x -q > gpurun_out/pdl2_pytest.log 2>&1; echo pytest pdl=1 rc=$?; tail -1 gpurun_out/pdl2_pytest.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pdl2_pytest_all.log 2>&1; echo pytest all rc=$?; tail -1 gpurun_out/pdl2_pytest_all.log
BENCH_ARGS="--config cfg1 --steps 300 --warmup 30" bash tools/ab.sh "" cur
bash tools/ab.sh "" cur
