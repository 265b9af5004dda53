# 4-GPU: repeated backward tests (flakiness check) + bench N=1, 2, 4 (peer transport)
mkdir -p gpurun_out
for i in 1 2 3; do timeout 300 python -m pytest tests/test_gpu_bwd.py tests/test_gpu_step.py -x -q 2>&1 | tail -1; done
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-e2e > gpurun_out/n1w.json 2> gpurun_out/n1w.err; echo n1 rc=$?
for N in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --steps 20 --warmup 3 --no-cpu > gpurun_out/n${N}w.json 2> gpurun_out/n${N}w.err; echo n$N rc=$?
done
python - <<PY
import json
for n in ("n1w","n2w","n4w"):
    try:
        d=json.loads(open(f"gpurun_out/{n}.json").read().strip().splitlines()[-1])
        print(n, round(d["ms_per_step"],3), round(d["value"]/1e6,2), "M/s", {k: round(v,3) for k,v in d.get("phases_ms",{}).items()})
    except Exception as e:
        print(n, "failed", e)
PY
tail -3 gpurun_out/n4w.err
