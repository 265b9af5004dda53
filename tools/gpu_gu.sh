# unique-row gradients: 256 positions per warp task (cur) vs 64 / 128 / 512 (wave tail vs per-task setup)
mkdir -p gpurun_out
RECD_LIB=build/variants/librecd_gu64.so timeout 600 python -m pytest tests/test_gpu_bwd.py tests/test_gpu_step.py -m gpu -x -q 2>&1 | tail -1
for rep in 1 2 3; do bash tools/ab.sh "" cur gu64 gu128 gu512; done
