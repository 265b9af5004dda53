mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
CUDA_VISIBLE_DEVICES=0 bash tools/ab.sh "" cur
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 20 --warmup 3 --no-cpu > gpurun_out/n2r.json 2> gpurun_out/n2r.err; echo n2 rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/n2r.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), round(d['value']/1e6,2), {k: round(v,3) for k,v in d['phases_ms'].items()})"
