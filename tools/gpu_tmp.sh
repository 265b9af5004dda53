timeout 900 python -m pytest tests/test_gpu_runs.py -x -q > gpurun_out/pytest_rv.log 2>&1
echo "pytest runs rc=$?"; tail -5 gpurun_out/pytest_rv.log
RECD_BWD_RUNS=1 timeout 900 python -m pytest tests/test_gpu_bwd.py tests/test_gpu_step.py tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest_rv2.log 2>&1
echo "pytest runs=1 rc=$?"; tail -5 gpurun_out/pytest_rv2.log
for rep in 1 2; do bash tools/ab_env.sh "" base; bash tools/ab_env.sh "RECD_BWD_RUNS=1" rv; done
RECD_BWD_RUNS=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" --csv --log-file gpurun_out/launches_rv.csv python bench.py --profile --steps 1 --warmup 1 --no-cpu --no-graph > gpurun_out/launches_rv.log 2>&1; echo launches rc=$?
python profiles/launches_summary.py gpurun_out/launches_rv.csv > gpurun_out/launches_rv.txt 2>&1; head -40 gpurun_out/launches_rv.txt
