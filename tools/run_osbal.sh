RECD_LIB=build/variants/librecd_osbal.so timeout 300 python -m pytest tests/test_gpu_sort.py tests/test_gpu_bwd.py -x -q 2>&1 | tail -2
bash tools/ab.sh "" cur osbal
