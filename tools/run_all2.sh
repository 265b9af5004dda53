mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 600 python bench.py > gpurun_out/n1.json 2> gpurun_out/n1.err; echo rc=$?
tail -c 1500 gpurun_out/n1.json
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 > gpurun_out/n2.json 2> gpurun_out/n2.err; echo rc=$?
python - <<PY
import json
for n in ("n1","n2"):
    d=json.loads(open(f"gpurun_out/{n}.json").read().strip().splitlines()[-1])
    print(n, d["ms_per_step"], d["value"], d["e2e"], d.get("gpu_launches_per_step"))
PY
