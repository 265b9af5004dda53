mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "sharded or peer or dist or deferred" > gpurun_out/pytest_r2h.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_r2h.log
timeout 900 python bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/bench_r2h_n2.json 2> gpurun_out/bench_r2h_n2.err; echo bench n2 rc=$?
tail -c 300 gpurun_out/bench_r2h_n2.err
python -c "
import json
d=json.loads(open('gpurun_out/bench_r2h_n2.json').read().strip().splitlines()[-1])
print('n', d['n_gpus'], 'ms', d['ms_per_step'], 'value', d['value'], 'roof', d['roofline']['frac'], 'step', d['step_roofline']['frac'], 'e2e', d['e2e']['value'])
"
CUDA_VISIBLE_DEVICES=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" --csv --log-file gpurun_out/launches_cfg1.csv python bench.py --config cfg1 --profile --steps 1 --warmup 1 --no-cpu --no-graph > gpurun_out/launches_cfg1.log 2>&1; echo launches rc=$?
python profiles/launches_summary.py gpurun_out/launches_cfg1.csv 2>&1 | head -30
