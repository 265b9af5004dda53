# 2-GPU: sharded parity tests + bench N=2 with and without the owner-side overlap
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_sharded.py -m gpu -x -q > gpurun_out/pytest_sharded2.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_sharded2.log
for O in "" "--no-overlap"; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 20 --warmup 3 --no-cpu $O > gpurun_out/n2o$O.json 2> gpurun_out/n2o$O.err; echo n2 $O rc=$?
python - <<PY
import json
d=json.loads(open("gpurun_out/n2o$O.json").read().strip().splitlines()[-1])
print("$O", d["ms_per_step"], d["value"], {k: round(v,3) for k,v in d.get("phases_ms",{}).items()})
PY
done
