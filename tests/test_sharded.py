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

from paper_2211_05239_b200.sharded import auto_shards, place_pairs, plan_exchange, shard_rows

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_shard_rows_partition():
    for rows in (1, 7, 1000, 10_000_000):
        for R in (1, 2, 3, 4, 8):
            sizes = [shard_rows(rows, R, r) for r in range(R)]
            assert sum(sizes) == rows
            assert sizes == [len(range(r, rows, R)) for r in range(R)]


def test_place_pairs_lpt():
    # equal weights spread evenly; heavy pairs go to distinct ranks
    assert sorted(place_pairs([1.0] * 8, 4)) == [0, 0, 1, 1, 2, 2, 3, 3]
    pl = place_pairs([10.0, 10.0, 1.0, 1.0, 1.0, 1.0], 2)
    assert pl[0] != pl[1]
    load = [0.0, 0.0]
    for p, r in enumerate(pl):
        load[r] += [10.0, 10.0, 1.0, 1.0, 1.0, 1.0][p]
    assert load == [12.0, 12.0]
    assert place_pairs([3.0, 1.0, 2.0], 1) == [0, 0, 0]
    assert place_pairs([5.0, 5.0], 4) == [0, 1]   # deterministic tie-break


def test_auto_shards():
    gb = 1 << 30
    assert auto_shards([1.0] * 26, [5 * gb] * 26, 8, 100 * gb) == 1      # cfg2 tables fit whole
    assert auto_shards([1.0] * 4, [60 * gb] * 4, 8, 100 * gb) == 1       # one table per rank
    assert auto_shards([1.0] * 2, [300 * gb] * 2, 8, 100 * gb) == 3      # must split: 6 x 100 GB
    with pytest.raises(ValueError):
        auto_shards([1.0], [2000 * gb], 8, 100 * gb)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    F, S = 3, 3                                   # more shards than ranks
    P = F * S
    place = place_pairs([float(1 + p // S) for p in range(P)], world)
    rng = np.random.default_rng(rank)
    ids = rng.integers(0, 50, size=P)             # this rank's IDs per (table, shard)
    urows = np.repeat(rng.integers(1, 20, size=F), S)
    mask = (np.array(place)[None, :] == np.arange(world)[:, None]).astype(np.int64)
    send = np.concatenate([mask * ids[None, :], mask * urows[None, :]], axis=1)
    recv = torch.zeros((world, 2 * P), dtype=torch.int64)
    dist.all_to_all_single(recv, torch.from_numpy(send))
    pl = plan_exchange(send, recv.numpy())
    ok = bool((pl.send_ids == ids).all() and (pl.send_rows == urows).all())
    for p in range(P):
        if place[p] != rank:
            ok &= pl.owner_rows(p) == 0 and pl.owner_ids(p) == 0
        ok &= pl.recv_id_base(p, world - 1) + pl.recv_ids[world - 1, p] == pl.owner_ids(p)
        ok &= pl.recv_row_base(p, world - 1) + pl.recv_rows[world - 1, p] == pl.owner_rows(p)
    # global conservation: IDs / rows sent == received
    tot = torch.tensor([int(ids.sum()), int(pl.recv_ids.sum()),
                        int(urows.sum()), int(pl.recv_rows.sum())], dtype=torch.int64)
    dist.all_reduce(tot)
    ok &= int(tot[0]) == int(tot[1]) and int(tot[2]) == int(tot[3])
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
@pytest.mark.parametrize("transport,op,shards", [
    ("nccl", "sum", 2), ("nccl", "avg", 2), ("nccl", "sum", 1), ("nccl", "sum", 3),
    ("peer", "sum", 2), ("peer", "avg", 2), ("peer", "sum", 1), ("peer", "sum", 3)])
def test_sharded_step_two_gpus(transport, op, shards):
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs (gpurun --gpus 2)")
    env = dict(os.environ, POOL_OP=op, SHARDS=str(shards), TRANSPORT=transport)
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node=2", "--master-addr=127.0.0.1",
                        f"--master-port={29600 + os.getpid() % 1000}",
                        os.path.join(ROOT, "tests", "dist_sharded_check.py")],
                       capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
