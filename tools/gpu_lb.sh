# one-sweep look-back after early publication: interleaved tickets (il), 16- / 4-deep look-back vs 8 (cur)
mkdir -p gpurun_out
RECD_LIB=build/variants/librecd_il.so timeout 900 python -m pytest tests/test_gpu_sort.py tests/test_gpu_bwd.py tests/test_gpu_step.py -m gpu -x -q > gpurun_out/lb_pytest.log 2>&1; echo pytest il rc=$?; tail -1 gpurun_out/lb_pytest.log
for rep in 1 2 3; do bash tools/ab.sh "" cur il lb16 lb4; done
BENCH_ARGS="--config cfg1 --steps 300 --warmup 30" bash tools/ab.sh "" cur il
