# k_copy: 8 gathers in flight per thread (cur) vs 4 (cpilp4); block -> feature by binary search (both)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/cp_pytest.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/cp_pytest.log
for rep in 1 2 3; do bash tools/ab.sh "" cur cpilp4; done
BENCH_ARGS="--config cfg1 --steps 300 --warmup 30" bash tools/ab.sh "" cur cpilp4
