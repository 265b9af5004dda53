bash tools/ab.sh "not sharded" cur gpk1
BENCH_ARGS=--no-overlap bash tools/ab.sh "" cur
timeout 600 python -m pytest tests -m gpu -x -q -k sharded > gpurun_out/pytest_sharded.log 2>&1; echo sharded rc=$?; tail -2 gpurun_out/pytest_sharded.log
