# 4-GPU verification at HEAD: full GPU suite (sharded tests run), cfg5-scale parity on 4 ranks,
# bench.py --gpus 2 / 4 self-launched (S auto) and N=4 row-sharded S=4
mkdir -p gpurun_out
T=${1:-m4}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$T.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_$T.log
SCALE=cfg5 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 --master-port=29733 tests/dist_sharded_check.py > gpurun_out/dist_cfg5_$T.log 2>&1; echo dist cfg5 rc=$?
grep '"rank"' gpurun_out/dist_cfg5_$T.log | head -4
for cfg in "2 0" "4 0" "4 4"; do
  set -- $cfg
  timeout 900 python bench.py --gpus $1 --steps 20 --warmup 5 --shards $2 > gpurun_out/bench_${T}_n$1_s$2.json 2> gpurun_out/bench_${T}_n$1_s$2.err; echo bench n$1 S=$2 rc=$?
  python -c "
import json
d=json.loads(open('gpurun_out/bench_${T}_n$1_s$2.json').read().strip().splitlines()[-1])
print('n', d['n_gpus'], 'ms', round(d['ms_per_step'],3), 'M/s', round(d['value']/1e6,2), 'S', d['sharding']['shards_per_table'], 'roof', round(d['roofline']['frac'],3), 'step', round(d['step_roofline']['frac'],3), 'e2e', (d.get('e2e') or {}).get('value'))
print(' phases', {k: round(v, 3) for k, v in d['phases_ms'].items()})
"
done
