mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_graph_batches.py tests/test_gpu_step.py tests/test_gpu_dedup.py tests/test_gpu_bwd.py -m gpu -x -q > gpurun_out/pytest_r2e.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_r2e.log
for extra in "" "--no-pipeline"; do
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu $extra > gpurun_out/bench_r2e$extra.json 2> gpurun_out/bench_r2e$extra.err; echo bench $extra rc=$?
tail -c 300 gpurun_out/bench_r2e$extra.err
python -c "
import json
d=json.loads(open('gpurun_out/bench_r2e$extra.json').read().strip().splitlines()[-1])
print('ms', d['ms_per_step'], 'value', d['value'], 'roof', d['roofline']['frac'], 'step', d['step_roofline']['frac'], 'launches', d['gpu_launches_per_step'])
print(' e2e', d['e2e']['value'], d['e2e']['ms_per_step'])
"
done
