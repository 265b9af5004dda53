mkdir -p gpurun_out
for S in 1 2 4; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 4 --steps 20 --warmup 3 --shards $S --no-cpu > gpurun_out/n4_peer_s$S.json 2> gpurun_out/n4_peer_s$S.err; echo rc=$?
python - <<PY
import json; d=json.loads(open("gpurun_out/n4_peer_s$S.json").read().strip().splitlines()[-1])
print($S, d["ms_per_step"], d["value"], d["gpu_launches_per_step"], {k: round(v,3) for k,v in d["phases_ms"].items()})
PY
done
