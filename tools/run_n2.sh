set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_sharded.py -m gpu -x -q 2>&1 | tail -15
for S in 2 1; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 20 --warmup 3 --shards $S --no-cpu > gpurun_out/n2_s$S.json 2> gpurun_out/n2_s$S.err; echo rc=$?
tail -c 3000 gpurun_out/n2_s$S.json
done
