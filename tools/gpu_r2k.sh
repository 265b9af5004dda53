mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "not sharded and not peer and not dist" > gpurun_out/pytest_r2k.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_r2k.log
bash tools/ab.sh "" cur cur
BENCH_ARGS="--config cfg1 --steps 200" bash tools/ab.sh "" cur
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" --csv --log-file gpurun_out/launches_cfg1b.csv python bench.py --config cfg1 --profile --steps 1 --warmup 1 --no-cpu --no-graph > gpurun_out/launches_cfg1b.log 2>&1; echo launches rc=$?
python profiles/launches_summary.py gpurun_out/launches_cfg1b.csv 2>&1 | head -14
