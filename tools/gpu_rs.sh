# row scan: stepped rows (no per-pair division) -- parity + A/B vs the thread-contiguous scan
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_dedup.py tests/test_gpu_step.py tests/test_gpu_graph_batches.py tests/test_gpu_fullsize.py tests/test_gpu_pool.py tests/test_gpu_stats.py -m gpu -x -q > gpurun_out/rs_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/rs_pytest.log
for rep in 1 2 3; do bash tools/ab.sh "" cur nocoal; done
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:"k_rowscan" --csv --log-file gpurun_out/rs_ncu.csv python bench.py --profile --steps 1 --warmup 1 --no-cpu --no-graph > gpurun_out/rs_ncu.log 2>&1; echo ncu rc=$?
grep -h "k_rowscan" gpurun_out/rs_ncu.csv | awk -F'","' '{print $13, $15}' | head -4
