"""Row-sharded multi-GPU path: host logic on CPU (gloo, world_size 2) and the
GPU parity script under torchrun when >= 2 GPUs are visible."""

import os
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2211_05239_b200.sharded import plan_exchange, shard_rows

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_shard_rows_partition():
    for rows in (1, 7, 1000, 10_000_000):
        for R in (1, 2, 3, 4, 8):
            sizes = [shard_rows(rows, R, r) for r in range(R)]
            assert sum(sizes) == rows
            assert sizes == [len(range(r, rows, R)) for r in range(R)]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    F = 3
    rng = np.random.default_rng(rank)
    send = np.zeros((world, 2 * F), np.int64)
    send[:, :F] = rng.integers(0, 50, size=(world, F))      # IDs for owner o
    send[:, F:] = rng.integers(1, 20, size=F)[None, :]      # unique rows (same for every owner)
    gathered = [torch.zeros((world, 2 * F), dtype=torch.int64) for _ in range(world)]
    dist.all_gather(gathered, torch.from_numpy(send))
    recv = np.stack([gathered[s].numpy()[rank] for s in range(world)])  # what all_to_all delivers
    pl = plan_exchange(send, recv)
    ok = True
    for f in range(F):
        # bases are prefix sums, owner totals are the sums
        ok &= pl.recv_id_base(f, world - 1) + pl.recv_ids[world - 1, f] == pl.owner_ids(f)
        ok &= pl.owner_rows(f) == sum(gathered[s].numpy()[rank][F + f] for s in range(world))
        ok &= pl.send_id_base(f, world - 1) + pl.send_ids[world - 1, f] == send[:, f].sum()
    # global conservation: IDs sent == IDs received
    tot = torch.tensor([int(send[:, :F].sum()), int(pl.recv_ids.sum())], dtype=torch.int64)
    dist.all_reduce(tot)
    ok &= int(tot[0]) == int(tot[1])
    q.put(bool(ok))
    dist.destroy_process_group()


def test_exchange_plan_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert all(q.get(timeout=5) for _ in procs)


@pytest.mark.gpu
@pytest.mark.parametrize("op", ["sum", "avg"])
def test_sharded_step_two_gpus(op):
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs (gpurun --gpus 2)")
    env = dict(os.environ, POOL_OP=op)
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node=2", "--master-addr=127.0.0.1",
                        f"--master-port={29600 + os.getpid() % 1000}",
                        os.path.join(ROOT, "tests", "dist_sharded_check.py")],
                       capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
