# usage (GPU box): tools/ab_var_tests.sh v1 v2 ... -- backward/step tests on each variant library
for v in "$@"; do
  RECD_LIB=build/variants/librecd_$v.so timeout 600 python -m pytest tests/test_gpu_bwd.py tests/test_gpu_step.py -m gpu -x -q > gpurun_out/vt_$v.log 2>&1
  echo "$v tests rc=$?"; tail -1 gpurun_out/vt_$v.log
done
