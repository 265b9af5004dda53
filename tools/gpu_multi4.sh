# usage (GPU box, 4 GPUs): tools/gpu_multi4.sh <tag>
mkdir -p gpurun_out
T=$1
nvidia-smi nvlink -h > gpurun_out/nvlink_help_$T.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "sharded or peer or dist" > gpurun_out/pytest_$T.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_$T.log
SCALE=cfg5 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 --master-port=29733 tests/dist_sharded_check.py > gpurun_out/dist_cfg5_$T.log 2>&1; echo dist cfg5 rc=$?
grep '"rank"' gpurun_out/dist_cfg5_$T.log
for S in 0 4; do
  timeout 900 python bench.py --gpus 4 --steps 20 --warmup 5 --shards $S > gpurun_out/bench_${T}_n4_s$S.json 2> gpurun_out/bench_${T}_n4_s$S.err; echo bench n4 S=$S rc=$?
  tail -c 300 gpurun_out/bench_${T}_n4_s$S.err
  python -c "
import json
d=json.loads(open('gpurun_out/bench_${T}_n4_s$S.json').read().strip().splitlines()[-1])
print('n', d['n_gpus'], 'ms', d['ms_per_step'], 'value', d['value'], 'S', d['sharding']['shards_per_table'], 'roof', d['roofline']['frac'], 'step', d['step_roofline']['frac'], 'e2e', (d['e2e'] or {}).get('value'))
print(' phases', {k: round(v, 3) for k, v in d['phases_ms'].items()})
"
done
# NVLink bytes of the N=2 step: link counters around two runs that differ only in timed steps
for st in 20 220; do
  nvidia-smi nvlink -gt d > gpurun_out/nvl_${T}_before_$st.txt 2>&1
  CUDA_VISIBLE_DEVICES=0,1 timeout 900 python bench.py --gpus 2 --steps $st --warmup 5 --no-e2e > gpurun_out/bench_${T}_n2_st$st.json 2> gpurun_out/bench_${T}_n2_st$st.err
  echo "n2 steps=$st rc=$?"
  nvidia-smi nvlink -gt d > gpurun_out/nvl_${T}_after_$st.txt 2>&1
done
head -30 gpurun_out/nvl_${T}_after_220.txt
