# GPU box: ballot digit matching in the sort (variant osb) vs match_any
RECD_LIB=build/variants/librecd_osb.so timeout 600 python -m pytest tests/test_gpu_sort.py tests/test_gpu_bwd.py -x -q > gpurun_out/vt_osb.log 2>&1; echo "osb tests rc=$?"; tail -1 gpurun_out/vt_osb.log
RECD_SORT_SPLIT=1 RECD_LIB=build/variants/librecd_osb.so timeout 600 python -m pytest tests/test_gpu_sort.py -x -q > gpurun_out/vt_osb2.log 2>&1; echo "osb split tests rc=$?"; tail -1 gpurun_out/vt_osb2.log
bash tools/ab.sh "" cur osb cur osb
export BENCH_ARGS="--rows 16777216 --dim 64"
for rep in 1 2; do
  RECD_LIB=build/variants/librecd_osb.so bash tools/ab_env.sh "RECD_SORT_SPLIT=1" osb_split24
  RECD_LIB=build/variants/librecd_osb.so bash tools/ab_env.sh "" osb_lsd24
done
