mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dedup.py tests/test_gpu_step.py tests/test_gpu_graph_batches.py tests/test_gpu_fullsize.py tests/test_gpu_partial.py tests/test_gpu_transforms.py tests/test_gpu_encoder.py -m gpu -x -q > gpurun_out/pytest_r2i.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_r2i.log
bash tools/ab.sh "" cur cur
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" --csv --log-file gpurun_out/launches_r2i.csv python bench.py --profile --steps 1 --warmup 1 --no-cpu --no-graph > gpurun_out/launches_r2i.log 2>&1; echo launches rc=$?
python profiles/launches_summary.py gpurun_out/launches_r2i.csv 2>&1 | head -16
timeout 900 python bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/bench_r2i_n2.json 2> gpurun_out/bench_r2i_n2.err; echo bench n2 rc=$?
tail -c 300 gpurun_out/bench_r2i_n2.err
python -c "
import json
d=json.loads(open('gpurun_out/bench_r2i_n2.json').read().strip().splitlines()[-1])
print('n', d['n_gpus'], 'ms', d['ms_per_step'], 'value', d['value'], 'roof', d['roofline']['frac'], 'step', d['step_roofline']['frac'], 'e2e', d['e2e']['value'])
"
