# 4-GPU verification of the final state: full GPU suite (multi-GPU tests
# included), row-sharded parity on 4 GPUs, bench N=2 / N=4 (both arms)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu4.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu4.log
for N in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --steps 30 --warmup 5 > gpurun_out/n${N}f.json 2> gpurun_out/n${N}f.err; echo n$N rc=$?
tail -c 600 gpurun_out/n${N}f.json
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 4 --steps 2 --warmup 3 > gpurun_out/ref4f.json 2> gpurun_out/ref4f.err; echo ref4 rc=$?
tail -c 400 gpurun_out/ref4f.json
bash tools/run_dist4.sh
