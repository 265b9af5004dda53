# sort state cleared in k_os_setup (cur) vs two memset nodes (memset)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/clr_pytest.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/clr_pytest.log
for rep in 1 2 3; do BENCH_ARGS="--config cfg1 --steps 300 --warmup 30" bash tools/ab.sh "" cur memset; done
for rep in 1 2; do bash tools/ab.sh "" cur memset; done
