mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_graph_batches.py tests/test_gpu_stats.py tests/test_table_init.py tests/test_gpu_fullsize.py tests/test_gpu_step.py -m gpu -x -q > gpurun_out/pytest_r2b.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/pytest_r2b.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_r2b.json 2> gpurun_out/bench_r2b.err; echo bench rc=$?
tail -c 600 gpurun_out/bench_r2b.err
timeout 600 python bench.py --config cfg1 --steps 200 --warmup 20 > gpurun_out/bench_r2b_cfg1.json 2> gpurun_out/bench_r2b_cfg1.err; echo cfg1 rc=$?
tail -c 600 gpurun_out/bench_r2b_cfg1.err
for f in gpurun_out/bench_r2b.json gpurun_out/bench_r2b_cfg1.json; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f ms', d['ms_per_step'], 'value', d['value'], 'launches', d['gpu_launches_per_step'])
print(' roof', d['roofline']['kernel'], d['roofline']['frac'], 'step', d['step_roofline']['frac'], d['phases_ms'])
print(' e2e', d['e2e'], 'cpu', d['cpu_baseline'])
"; done
