mkdir -p gpurun_out
for N in 8; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --steps 20 --warmup 3 --no-cpu > gpurun_out/n${N}z.json 2> gpurun_out/n${N}z.err; echo n$N rc=$?
done
python - <<PY
import json
for n in ("n8z",):
    try:
        d=json.loads(open(f"gpurun_out/{n}.json").read().strip().splitlines()[-1])
        print(n, round(d["ms_per_step"],3), round(d["value"]/1e6,2), "M/s", {k: round(v,3) for k,v in d.get("phases_ms",{}).items()})
    except Exception as e:
        print(n, "failed", e)
PY
tail -3 gpurun_out/n8z.err
