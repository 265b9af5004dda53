mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_runs.py -m gpu -x -q > gpurun_out/pytest_runs2a.log 2>&1; echo pytest runs rc=$?; tail -3 gpurun_out/pytest_runs2a.log
RECD_BWD_RUNS=1 timeout 900 python -m pytest tests/test_gpu_bwd.py tests/test_gpu_step.py tests/test_gpu_graph_batches.py tests/test_gpu_fullsize.py -m gpu -x -q > gpurun_out/pytest_runs2b.log 2>&1; echo pytest runs=1 rc=$?; tail -3 gpurun_out/pytest_runs2b.log
for R in 0 1 0 1; do bash tools/ab_env.sh "RECD_BWD_RUNS=$R" runs$R; done
RECD_BWD_RUNS=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" --csv --log-file gpurun_out/launches_runs2.csv python bench.py --profile --steps 1 --warmup 1 --no-cpu --no-graph > gpurun_out/launches_runs2.log 2>&1; echo launches rc=$?
python profiles/launches_summary.py gpurun_out/launches_runs2.csv 2>&1 | head -24
