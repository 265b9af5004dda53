# one-sweep first pass: early publication in pass 0 (cur) vs late (late0); 4-deep look-back with interleaving (lb4il)
mkdir -p gpurun_out
RECD_LIB=build/variants/librecd_late0.so timeout 900 python -m pytest tests/test_gpu_sort.py tests/test_gpu_bwd.py -m gpu -x -q > gpurun_out/p0_pytest.log 2>&1; echo pytest late0 rc=$?; tail -1 gpurun_out/p0_pytest.log
for rep in 1 2 3; do bash tools/ab.sh "" cur late0 lb4il; done
for v in cur late0; do
  lib=paper_2211_05239_b200/librecd.so; [ $v != cur ] && lib=build/variants/librecd_$v.so
  RECD_LIB=$lib timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_onesweep" --csv --log-file gpurun_out/p0_ncu_$v.csv python bench.py --profile --steps 1 --warmup 1 --no-cpu --no-graph > gpurun_out/p0_ncu_$v.log 2>&1; echo ncu $v rc=$?
  grep -h "gpu__time" gpurun_out/p0_ncu_$v.csv | awk -F'","' '{print $15}' | tr -d '"' | head -10 | tr '\n' ' '; echo
done
