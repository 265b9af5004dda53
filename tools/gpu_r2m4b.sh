# 4-GPU bench at HEAD: sharded tests, bench.py --gpus 2 / 4 self-launched (S auto)
mkdir -p gpurun_out
T=${1:-m4b}
timeout 900 python -m pytest tests/test_sharded.py -m gpu -x -q > gpurun_out/pytest_$T.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_$T.log
for N in 2 4; do
  timeout 900 python bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/bench_${T}_n$N.json 2> gpurun_out/bench_${T}_n$N.err; echo bench n$N rc=$?
  python -c "
import json
d=json.loads(open('gpurun_out/bench_${T}_n$N.json').read().strip().splitlines()[-1])
print('n', d['n_gpus'], 'ms', round(d['ms_per_step'],3), 'M/s', round(d['value']/1e6,2), 'S', d['sharding']['shards_per_table'], 'roof', round(d['roofline']['frac'],3), 'step', round(d['step_roofline']['frac'],3), 'e2e', (d.get('e2e') or {}).get('value'))
print(' phases', {k: round(v, 3) for k, v in d['phases_ms'].items()})
"
done
