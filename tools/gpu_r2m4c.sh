# 4-GPU box at final HEAD: the whole GPU suite (sharded tests included) + cfg5-scale parity on 4 ranks
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_m4c.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_m4c.log
SCALE=cfg5 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 --master-port=29733 tests/dist_sharded_check.py > gpurun_out/dist_cfg5_m4c.log 2>&1; echo dist cfg5 rc=$?
grep '"rank"' gpurun_out/dist_cfg5_m4c.log | head -4
