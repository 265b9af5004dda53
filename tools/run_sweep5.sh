mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bwd.py tests/test_gpu_pool.py -m gpu -x -q > gpurun_out/t.log 2>&1; echo tests rc=$?
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/var_main.json 2>&1; echo main rc=$?
bash tools/sweep.sh prev
python tools/show_var.py main prev
for v in main prev; do python - <<PY
import json; d=json.loads(open("gpurun_out/var_$v.json").read().strip().splitlines()[-1]); print("$v", {k: (round(x["ms"],3), round(x["achieved_gbs"])) for k,x in d["kernels"].items()})
PY
done
tail -2 gpurun_out/t.log
