set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_sharded.py -m gpu -x -q -k peer 2>&1 | tail -30
for T in peer; do for S in 2 1; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 20 --warmup 3 --shards $S --transport $T --no-cpu > gpurun_out/n2_${T}_s$S.json 2> gpurun_out/n2_${T}_s$S.err; echo rc=$?
tail -c 2500 gpurun_out/n2_${T}_s$S.json; tail -5 gpurun_out/n2_${T}_s$S.err
done; done
