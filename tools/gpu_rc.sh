# scatter: 256 sorted positions per warp task (cur) vs 128 / 384
mkdir -p gpurun_out
for v in rc128 rc384; do RECD_LIB=build/variants/librecd_$v.so timeout 600 python -m pytest tests/test_gpu_bwd.py tests/test_gpu_step.py tests/test_gpu_fullsize.py -m gpu -x -q 2>&1 | tail -1; done
for rep in 1 2 3; do bash tools/ab.sh "" cur rc128 rc384; done
