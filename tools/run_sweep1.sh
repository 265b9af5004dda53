mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pool.py tests/test_gpu_bwd.py -m gpu -x -q 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/var_main.json 2>&1; echo main rc=$?
bash tools/sweep.sh base noring l2_0 l2_2 k8m4 k12m3 k24m2
python tools/show_var.py main base noring l2_0 l2_2 k8m4 k12m3 k24m2
for v in main base; do python - <<PY
import json; d=json.loads(open("gpurun_out/var_$v.json").read().strip().splitlines()[-1]); print("$v", {k: (round(x["ms"],3), round(x["achieved_gbs"])) for k,x in d["kernels"].items()})
PY
done
