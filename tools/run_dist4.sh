# 4-GPU parity of the row-sharded step against the oracle (tests/dist_sharded_check.py)
mkdir -p gpurun_out
for cfg in "peer sum 1" "peer avg 4" "peer sum 3" "nccl sum 1" "nccl avg 2"; do
  set -- $cfg
  TRANSPORT=$1 POOL_OP=$2 SHARDS=$3 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 \
    --master-addr 127.0.0.1 --master-port 29533 tests/dist_sharded_check.py > gpurun_out/dist4_$1_$2_$3.log 2>&1
  echo "$cfg rc=$?"; grep -h '"rank"' gpurun_out/dist4_$1_$2_$3.log | head -4
done
