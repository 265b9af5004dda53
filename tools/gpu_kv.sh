# one-sweep 64-bit (key, value) staging (cur) vs two 32-bit arrays (kv32): parity, sort probe, step A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sort.py tests/test_gpu_bwd.py tests/test_gpu_step.py tests/test_gpu_runs.py tests/test_gpu_jagged.py -m gpu -x -q > gpurun_out/kv_pytest.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/kv_pytest.log
timeout 600 python tools/sort_probe.py
RECD_LIB=build/variants/librecd_kv32.so timeout 600 python tools/sort_probe.py
for rep in 1 2 3; do bash tools/ab.sh "" cur kv32; done
