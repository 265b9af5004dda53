mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bwd.py tests/test_gpu_step.py tests/test_gpu_graph_batches.py tests/test_gpu_fullsize.py tests/test_gpu_sort.py -m gpu -x -q > gpurun_out/pytest_runs.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/pytest_runs.log
for R in 1 0 1 0; do
RECD_BWD_RUNS=$R timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/bench_runs$R.json 2> gpurun_out/bench_runs$R.err; echo bench runs=$R rc=$?
tail -c 300 gpurun_out/bench_runs$R.err
python -c "
import json
d=json.loads(open('gpurun_out/bench_runs$R.json').read().strip().splitlines()[-1])
print('runs=$R ms', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phases_ms'].items()}, {k: round(v['ms'],3) for k, v in d['kernels'].items()})
"
done
RECD_BWD_RUNS=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" --csv --log-file gpurun_out/launches_runs.csv python bench.py --profile --steps 1 --warmup 1 --no-cpu --no-graph > gpurun_out/launches_runs.log 2>&1; echo launches rc=$?
python profiles/launches_summary.py gpurun_out/launches_runs.csv 2>&1 | head -30
