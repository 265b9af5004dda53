# usage (GPU box, N GPUs): tools/gpu_multi.sh <tag> <N>  -- N-GPU tests + bench S=auto and S=N
mkdir -p gpurun_out
N=$2
timeout 900 python -m pytest tests -m gpu -x -q -k "sharded or peer or dist" > gpurun_out/pytest_$1.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_$1.log
timeout 900 python bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/bench_$1_auto.json 2> gpurun_out/bench_$1_auto.err; echo bench auto rc=$?
tail -c 400 gpurun_out/bench_$1_auto.err
timeout 900 python bench.py --gpus $N --steps 20 --warmup 5 --shards $N --no-e2e > gpurun_out/bench_$1_sN.json 2> gpurun_out/bench_$1_sN.err; echo bench sN rc=$?
tail -c 400 gpurun_out/bench_$1_sN.err
for f in gpurun_out/bench_$1_auto.json gpurun_out/bench_$1_sN.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', 'n', d['n_gpus'], 'ms', d['ms_per_step'], 'value', d['value'], 'S', d['sharding']['shards_per_table'])
print(' roof', d['roofline']['frac'], 'step', d['step_roofline']['frac'], d['step_roofline']['per_rank_frac'])
print(' phases', d['phases_ms'])
print(' e2e', d['e2e']['value'] if d.get('e2e') else None)
"; done
