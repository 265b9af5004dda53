# shifted-window sharing in the pooled lookup (k_pool_win): parity, then cfg2 / cfg1 A/B vs the per-warp ring
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_pool.py tests/test_gpu_step.py tests/test_gpu_graph_batches.py tests/test_gpu_fullsize.py tests/test_gpu_dedup.py tests/test_gpu_encoder.py -m gpu -x -q > gpurun_out/win_pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/win_pytest.log
for rep in 1 2; do bash tools/ab.sh "" cur nowin; done
BENCH_ARGS="--config cfg1 --steps 300 --warmup 30" bash tools/ab.sh "" cur nowin
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none -k regex:"k_pool_(win|ring)" --csv --log-file gpurun_out/win_ncu.csv python bench.py --profile --steps 1 --warmup 1 --no-cpu --no-graph > gpurun_out/win_ncu.log 2>&1; echo ncu rc=$?
RECD_LIB=build/variants/librecd_nowin.so timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none -k regex:"k_pool_(win|ring)" --csv --log-file gpurun_out/win_ncu_off.csv python bench.py --profile --steps 1 --warmup 1 --no-cpu --no-graph > gpurun_out/win_ncu_off.log 2>&1; echo ncu off rc=$?
grep -h "k_pool" gpurun_out/win_ncu.csv gpurun_out/win_ncu_off.csv | cut -c1-400 | head -20
