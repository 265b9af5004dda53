# usage (GPU box): tools/gpu_quick.sh <tag> -- kernel tests + cfg2 bench line + launch list
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_sort.py tests/test_gpu_bwd.py tests/test_gpu_step.py tests/test_gpu_dedup.py tests/test_gpu_pool.py tests/test_gpu_graph_batches.py tests/test_gpu_jagged.py -m gpu -x -q > gpurun_out/pytest_$1.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_$1.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/bench_$1.json 2> gpurun_out/bench_$1.err; echo bench rc=$?
tail -c 300 gpurun_out/bench_$1.err
python -c "
import json
d=json.loads(open('gpurun_out/bench_$1.json').read().strip().splitlines()[-1])
print('ms', d['ms_per_step'], 'value', d['value'], 'roof', d['roofline']['kernel'], d['roofline']['frac'], 'step', d['step_roofline']['frac'])
print(' phases', d['phases_ms'], {k: v['ms'] for k, v in d['kernels'].items()})
"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" --csv --log-file gpurun_out/launches_$1.csv python bench.py --profile --steps 1 --warmup 1 --no-cpu --no-graph > gpurun_out/launches_$1.log 2>&1; echo launches rc=$?
python profiles/launches_summary.py gpurun_out/launches_$1.csv > gpurun_out/launches_$1.txt 2>&1; head -14 gpurun_out/launches_$1.txt
