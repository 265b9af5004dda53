# GPU box: split sort (top pass + shared-memory bucket sort) -- tests and A/B
timeout 900 python -m pytest tests/test_gpu_sort.py tests/test_gpu_bwd.py tests/test_gpu_step.py tests/test_gpu_runs.py tests/test_gpu_fullsize.py tests/test_gpu_graph_batches.py -x -q > gpurun_out/pytest_split.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_split.log
for rep in 1 2; do
  bash tools/ab_env.sh "RECD_SORT_SPLIT=0" lsd
  bash tools/ab_env.sh "" split
done
timeout 300 python tools/timeline.py --steps 10 > gpurun_out/tl_split.txt 2>&1; tail -8 gpurun_out/tl_split.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" --csv --log-file gpurun_out/launches_split.csv python bench.py --profile --steps 1 --warmup 1 --no-cpu --no-graph > gpurun_out/launches_split.log 2>&1; echo launches rc=$?
python profiles/launches_summary.py gpurun_out/launches_split.csv > gpurun_out/launches_split.txt 2>&1; head -30 gpurun_out/launches_split.txt
