# 2-GPU verification: full GPU test suite (incl. sharded parity), bench N=1 and N=2
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu2.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu2.log
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu > gpurun_out/n1v.json 2> gpurun_out/n1v.err; echo n1 rc=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 20 --warmup 3 --no-cpu > gpurun_out/n2v.json 2> gpurun_out/n2v.err; echo n2 rc=$?
python - <<PY
import json
for n in ("n1v","n2v"):
    try:
        d=json.loads(open(f"gpurun_out/{n}.json").read().strip().splitlines()[-1])
        print(n, d["ms_per_step"], d["value"], d.get("gpu_launches_per_step"), {k: round(v,3) for k,v in d.get("phases_ms",{}).items()})
    except Exception as e:
        print(n, "failed", e)
PY
tail -5 gpurun_out/n2v.err
