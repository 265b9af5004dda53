mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pool.py tests/test_gpu_bwd.py -m gpu -x -q > gpurun_out/t.log 2>&1; echo tests rc=$?
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/var_main.json 2>&1; echo main rc=$?
bash tools/sweep.sh noring nb1m3 nb3m2 nb4m1
python tools/show_var.py main noring nb1m3 nb3m2 nb4m1
tail -3 gpurun_out/t.log
