# A/B: coalesced uniform row scan (cur vs nocoal) on cfg2; small sort tiles (cur vs bigsort) on cfg1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sort.py tests/test_gpu_dedup.py tests/test_gpu_step.py tests/test_gpu_bwd.py tests/test_gpu_graph_batches.py tests/test_gpu_fullsize.py -m gpu -x -q > gpurun_out/w_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/w_pytest.log
for rep in 1 2; do bash tools/ab.sh "" cur nocoal; done
for rep in 1 2; do BENCH_ARGS="--config cfg1 --steps 200 --warmup 20" bash tools/ab.sh "" cur bigsort; done
