timeout 900 python -m pytest tests/test_gpu_rowcode.py tests/test_gpu_graph_batches.py -x -q > gpurun_out/pytest_rc.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_rc.log
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/bench_rc.json 2> gpurun_out/bench_rc.err; echo bench rc=$?
tail -3 gpurun_out/bench_rc.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_rc.json').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['e2e'])"
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu --e2e-wire raw > gpurun_out/bench_raw.json 2> gpurun_out/bench_raw.err; echo bench raw rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/bench_raw.json').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['e2e'])"
