# NCCL transport of the row-sharded step at HEAD (the north_star's all-to-all), N = 2 and 4, S auto
mkdir -p gpurun_out
for N in 2 4; do
  timeout 900 python bench.py --gpus $N --steps 20 --warmup 5 --transport nccl --no-e2e > gpurun_out/bench_nccl_n$N.json 2> gpurun_out/bench_nccl_n$N.err; echo bench nccl n$N rc=$?
  python -c "
import json
d=json.loads(open('gpurun_out/bench_nccl_n$N.json').read().strip().splitlines()[-1])
print('n', d['n_gpus'], 'ms', round(d['ms_per_step'],3), 'M/s', round(d['value']/1e6,2), d.get('sharding'), 'step', round(d['step_roofline']['frac'],3))
print(' phases', {k: round(v, 3) for k, v in d['phases_ms'].items()})
"
done
