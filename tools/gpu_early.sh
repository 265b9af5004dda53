# one-sweep sort: tile counts published before the ranking (cur) vs after (noearly): parity + A/B + sort launch times
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_sort.py tests/test_gpu_bwd.py tests/test_gpu_step.py tests/test_gpu_graph_batches.py tests/test_gpu_runs.py tests/test_gpu_fullsize.py tests/test_gpu_jagged.py tests/test_gpu_partial.py -m gpu -x -q > gpurun_out/ea_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/ea_pytest.log
for rep in 1 2 3; do bash tools/ab.sh "" cur early1 noearly; done
BENCH_ARGS="--config cfg1 --steps 300 --warmup 30" bash tools/ab.sh "" cur early1 noearly
for v in cur early1 noearly; do
  lib=paper_2211_05239_b200/librecd.so; [ $v != cur ] && lib=build/variants/librecd_$v.so
  RECD_LIB=$lib timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_onesweep|k_os_setup" --csv --log-file gpurun_out/ea_ncu_$v.csv python bench.py --profile --steps 1 --warmup 1 --no-cpu --no-graph > gpurun_out/ea_ncu_$v.log 2>&1; echo ncu $v rc=$?
  grep -h "gpu__time" gpurun_out/ea_ncu_$v.csv | awk -F'","' '{print $5, $15}' | cut -c1-120
done
