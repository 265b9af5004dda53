# usage (GPU box): tools/gpu_check.sh <tag>  -- GPU test suite + one default bench line
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_$1.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$1.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_$1.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$1.json 2> gpurun_out/bench_$1.err; echo bench rc=$?
tail -c 600 gpurun_out/bench_$1.err
python -c "
import json,sys
d=json.loads(open('gpurun_out/bench_$1.json').read().strip().splitlines()[-1])
print('ms', d['ms_per_step'], 'value', d['value'], 'phases', d.get('phases_ms'))
print('roof', d['roofline']['kernel'], d['roofline']['frac'], 'step', d['step_roofline']['frac'])
print('e2e', d['e2e']['value'] if d.get('e2e') else None, 'cpu', d['cpu_baseline'])
"
