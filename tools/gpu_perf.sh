# usage (GPU box): tools/gpu_perf.sh <tag> [ncu]  -- sort/bwd/step tests, cfg2 + cfg1 bench lines, optional ncu
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_sort.py tests/test_gpu_bwd.py tests/test_gpu_step.py tests/test_gpu_dedup.py tests/test_gpu_pool.py -m gpu -x -q > gpurun_out/pytest_$1.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_$1.log
for cfg in cfg2 cfg1; do
  st=20; [ $cfg = cfg1 ] && st=200
  timeout 600 python bench.py --config $cfg --steps $st --warmup 5 --no-cpu --no-e2e > gpurun_out/bench_$1_$cfg.json 2> gpurun_out/bench_$1_$cfg.err; echo bench $cfg rc=$?
  tail -c 300 gpurun_out/bench_$1_$cfg.err
  python -c "
import json
d=json.loads(open('gpurun_out/bench_$1_$cfg.json').read().strip().splitlines()[-1])
print('$cfg ms', d['ms_per_step'], 'value', d['value'], 'roof', d['roofline']['kernel'], d['roofline']['frac'], 'step', d['step_roofline']['frac'])
print(' phases', d['phases_ms'], {k: v['ms'] for k, v in d['kernels'].items()})
"
done
if [ "$2" = ncu ]; then bash tools/ncu_r2.sh $1; fi
