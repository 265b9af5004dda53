"""Multi-GPU parity check of the row-sharded step (run under torchrun).

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tests/dist_sharded_check.py

TRANSPORT=peer runs PeerShardedStep (NVLink peer memory, one CUDA-graph
replay), else ShardedTrainStep (NCCL).  Each rank deduplicates its contiguous chunk of one global session-clustered
batch; every table is split into S = $SHARDS (default R) shards id % S, the
(table, shard) pairs placed on ranks by the step's LPT placement.  Checked against the CPU
oracle (oracle/), on the same inputs:
  * dedup outputs (inverse, unique values/offsets): bit-exact
  * expanded pooled outputs: allclose(rtol=1e-5, atol=1e-5 * max|ref|)
  * updated tables (gathered from all shards) vs the oracle SGD over the whole
    global batch: same tolerance on the update.
Prints one JSON line per rank; exits 1 on a mismatch.
"""

import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import paper_2211_05239_b200 as R  # noqa: E402
from tools.datagen import (FeatureSpec, SampleCountDist, SessionConfig,  # noqa: E402
                                           generate_clustered_batch)
from paper_2211_05239_b200.peer import PeerShardedStep  # noqa: E402
from paper_2211_05239_b200.sharded import ShardedTrainStep  # noqa: E402


def close(a, b):
    scale = max(float(np.abs(b).max()), 1e-30)
    return bool(np.allclose(a, b, rtol=1e-5, atol=1e-5 * scale)), float(np.abs(a - b).max() / scale)


def main():
    op = os.environ.get("POOL_OP", "sum")
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    world, rank = dist.get_world_size(), dist.get_rank()
    B, D, rows, lr = 1500, 64, 3000, 0.05
    specs = [FeatureSpec("k0", "user_sequence", 4.0, rows, 0.3),
             FeatureSpec("k1", "user_sequence", 16.0, rows, 0.3),
             FeatureSpec("k2", "user_sequence", 40.0, rows, 0.3)]
    keys = [s.key for s in specs]
    cfg = SessionConfig(int(world * B / 6) + 50, SampleCountDist("geometric", 8.0), 0)
    chunks = [generate_clustered_batch(cfg, specs, B, row_start=r * B) for r in range(world)]
    mine = chunks[rank]
    full = {k: np.random.default_rng(100 + i).uniform(-0.1, 0.1, size=(rows, D)).astype(np.float32)
            for i, k in enumerate(keys)}
    S = int(os.environ.get("SHARDS", world))

    def make_table(k, j, n):
        w = torch.from_numpy(np.ascontiguousarray(full[k][j::S])).to(dev)
        assert w.shape[0] == n
        return R.EmbeddingTable(k, n, D, w)

    caps = {k: mine.values[k].size for k in keys}
    transport = os.environ.get("TRANSPORT", "nccl")
    cls = PeerShardedStep if transport == "peer" else ShardedTrainStep
    step = cls(keys, B, caps, {k: rows for k in keys}, D, make_table, op, lr, shards=S, device=dev)
    step.load_batch(mine.values, mine.offsets)
    grads = [np.random.default_rng(1000 * r + 7).standard_normal((B, D)).astype(np.float32)
             for r in range(world)]
    for g in step.grad_out:
        g.copy_(torch.from_numpy(grads[rank]))
    if transport == "peer":
        step.capture(warmup=False)   # one step, through the CUDA graph
        step.replay()
        torch.cuda.synchronize()
        step.check()
    else:
        step.run()
    torch.cuda.synchronize()

    res = {"rank": rank, "world": world, "shards": S, "transport": transport, "op": op, "ok": True,
           "pairs": step.mine}
    U, N = step.host_counts()
    # forward vs oracle on this rank's chunk
    worst_fwd = 0.0
    for f, k in enumerate(keys):
        inv, [(uv, uo)] = oracle.build_ikjt_arrays([(mine.values[k], mine.offsets[k])])
        same = (np.array_equal(step.inverse[f].cpu().numpy(), inv)
                and np.array_equal(step.uvalues[f][:N[f]].cpu().numpy(), uv)
                and np.array_equal(step.uoffsets[f][:U[f]].cpu().numpy(), uo))
        res["ok"] &= bool(same)
        ref = oracle.expand(oracle.pooled_lookup(uv, uo, full[k], op), inv)
        ok, err = close(step.out[f].cpu().numpy(), ref)
        res["ok"] &= ok
        worst_fwd = max(worst_fwd, err)
    res["fwd_max_rel_err"] = worst_fwd
    # backward: gather the shards, compare with the oracle SGD over all ranks
    worst_bwd = 0.0
    for f, k in enumerate(keys):
        # every row lives on exactly one rank: a sum over ranks reassembles the table
        new_t = torch.zeros((rows, D), device=dev)
        for p, t in step.tables.items():
            if p // S == f:
                new_t[p % S::S] = t.weights
        dist.all_reduce(new_t)
        new = new_t.cpu().numpy()
        g64 = np.zeros((rows, D), np.float64)
        for r in range(world):
            inv, [(uv, uo)] = oracle.build_ikjt_arrays([(chunks[r].values[k], chunks[r].offsets[k])])
            gu = oracle.pool_backward(grads[r], inv, uo.size)
            ids, gw = oracle.sparse_table_grad(gu, uv, uo, op)
            g64[ids] += gw
        delta_ref = -(np.float32(lr) * g64.astype(np.float32))
        ok, err = close(new - full[k], delta_ref)
        res["ok"] &= ok
        worst_bwd = max(worst_bwd, err)
    res["bwd_max_rel_err"] = worst_bwd
    res["launches"] = R.launch_count()
    print(json.dumps(res), flush=True)
    dist.destroy_process_group()
    return 0 if res["ok"] else 1


if __name__ == "__main__":
    sys.exit(main())
