# GPU box: split sort with uniform top digits (rows = 2^24, dim 64)
for rep in 1 2; do
  BENCH_ARGS="--rows 16777216 --dim 64" bash tools/ab_env.sh "RECD_SORT_SPLIT=0" lsd24
  BENCH_ARGS="--rows 16777216 --dim 64" bash tools/ab_env.sh "" split24
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" --csv --log-file gpurun_out/launches_split24.csv python bench.py --profile --steps 1 --warmup 1 --no-cpu --no-graph --rows 16777216 --dim 64 > gpurun_out/launches_split24.log 2>&1; echo launches rc=$?
python profiles/launches_summary.py gpurun_out/launches_split24.csv > gpurun_out/launches_split24.txt 2>&1; head -30 gpurun_out/launches_split24.txt
