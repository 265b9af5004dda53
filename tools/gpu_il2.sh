# full GPU suite at HEAD + interleaved tickets for multi-segment sorts (cur) vs none (noil)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/il2_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/il2_pytest.log
for rep in 1 2 3; do bash tools/ab.sh "" cur noil; done
BENCH_ARGS="--config cfg1 --steps 300 --warmup 30" bash tools/ab.sh "" cur noil
