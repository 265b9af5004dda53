# PDL A/B: GPU tests with PDL forced on (RECD_PDL=1, every step), then cfg1 / cfg2 bench with PDL off / auto / on
mkdir -p gpurun_out
RECD_PDL=1 timeout 900 python -m pytest tests/test_gpu_sort.py tests/test_gpu_dedup.py tests/test_gpu_pool.py tests/test_gpu_step.py tests/test_gpu_bwd.py tests/test_gpu_graph_batches.py tests/test_gpu_jagged.py tests/test_gpu_runs.py -m gpu -x -q > gpurun_out/pdl_pytest.log 2>&1; echo pytest pdl=1 rc=$?; tail -2 gpurun_out/pdl_pytest.log
for rep in 1 2; do
  BENCH_ARGS="--config cfg1 --steps 200 --warmup 20" bash tools/ab_env.sh "RECD_PDL=0" c1off
  BENCH_ARGS="--config cfg1 --steps 200 --warmup 20" bash tools/ab_env.sh "RECD_PDL_MAX=131072" c1on
done
bash tools/ab_env.sh "RECD_PDL=0" c2off
bash tools/ab_env.sh "RECD_PDL=1" c2on
bash tools/ab_env.sh "RECD_PDL=0" c2off
bash tools/ab_env.sh "RECD_PDL=1" c2on
