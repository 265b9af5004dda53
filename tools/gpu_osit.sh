# one-sweep tile size after early publication + interleaving: 16 items/thread (cur) vs 12, 20, 12 @ 4 CTAs/SM, 8 @ 5
mkdir -p gpurun_out
RECD_LIB=build/variants/librecd_os12.so timeout 600 python -m pytest tests/test_gpu_sort.py tests/test_gpu_bwd.py -m gpu -x -q 2>&1 | tail -1
RECD_LIB=build/variants/librecd_os20.so timeout 600 python -m pytest tests/test_gpu_sort.py tests/test_gpu_bwd.py -m gpu -x -q 2>&1 | tail -1
for rep in 1 2; do bash tools/ab.sh "" cur os12 os20 os12m4 os8m5; done
