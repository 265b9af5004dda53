mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bwd.py tests/test_gpu_pool.py tests/test_gpu_jagged.py -m gpu -x -q > gpurun_out/t.log 2>&1; echo tests rc=$?
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/var_main.json 2>&1; echo main rc=$?
bash tools/sweep.sh ct16 ct32 it16ct4 it16ct8 it12ct8
python tools/show_var.py main ct16 ct32 it16ct4 it16ct8 it12ct8
tail -3 gpurun_out/t.log
