mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dedup.py tests/test_gpu_step.py tests/test_gpu_graph_batches.py tests/test_gpu_fullsize.py tests/test_gpu_partial.py tests/test_gpu_stats.py -m gpu -x -q > gpurun_out/pytest_r2o.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_r2o.log
bash tools/ab.sh "" cur notma cur notma
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_rowscan" --csv --log-file gpurun_out/rowscan_r2o.csv python bench.py --profile --steps 1 --warmup 1 --no-cpu --no-graph > gpurun_out/rowscan_r2o.log 2>&1; echo ncu rc=$?
tail -4 gpurun_out/rowscan_r2o.csv
