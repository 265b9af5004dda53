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

SCALE=cfg5: the bench's multi-GPU workload instead -- 65,536 rows per rank,
the 26 cfg2 keys (lists up to 256), 10M x 128 tables -- with the oracle on
the touched rows of three sampled keys (lengths 8, 128, 256): the rows any
rank's batch touches are gathered from their owners before and after the
step into a compact table, the oracle pools / updates that.
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


def gather_rows(step, keys, f, ids, S, D, dev):
    """Rows `ids` of feature f's full table, from whichever rank owns each."""
    out = torch.zeros((ids.size, D), device=dev)
    tid = torch.as_tensor(ids, device=dev)
    for p, t in step.tables.items():
        if p // S == f:
            m = (tid % S) == (p % S)
            out[m] = t.weights[tid[m] // S]
    dist.all_reduce(out)
    return out.cpu().numpy()


def main_cfg5():
    from tools.datagen import cfg2_specs
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    world, rank = dist.get_world_size(), dist.get_rank()
    B, D, rows, lr = 65536, 128, 10_000_000, 0.05
    specs = cfg2_specs(rows)
    keys = [s.key for s in specs]
    nsess = int(np.ceil(B * world / 16.5 * 1.3)) + 64          # bench.make_batch
    cfg = SessionConfig(nsess, SampleCountDist("geometric", 16.5), 0)
    check = [0, 4, 5]
    # every spec: the generator draws all keys from one RNG stream per session
    chunks = {r: generate_clustered_batch(cfg, specs, B, row_start=r * B) for r in range(world)}
    mine = chunks[rank]
    S = int(os.environ.get("SHARDS", "1"))

    def make_table(k, j, n):
        return R.EmbeddingTable.create_on_device(f"{k}/shard{j}", n, D, seed=1000 * keys.index(k) + j,
                                                 device=dev)

    caps = {k: mine.values[k].size for k in keys}
    step = PeerShardedStep(keys, B, caps, {k: rows for k in keys}, D, make_table, "sum", lr,
                           shards=S, device=dev)
    step.load_batch(mine.values, mine.offsets)
    grads = {f: [np.random.default_rng(1000 * r + 7 + f).standard_normal((B, D)).astype(np.float32)
                 for r in range(world)] for f in check}
    step.fill_grad_out(5)
    for f in check:
        step.grad_out[f].copy_(torch.from_numpy(grads[f][rank]))
    ikjts = {(r, f): oracle.build_ikjt_arrays([(chunks[r].values[keys[f]], chunks[r].offsets[keys[f]])])
             for r in range(world) for f in check}
    ids = {f: np.unique(np.concatenate([ikjts[(r, f)][1][0][0] for r in range(world)])) for f in check}
    w0 = {f: gather_rows(step, keys, f, ids[f], S, D, dev) for f in check}
    step.capture(warmup=False)
    step.replay()
    torch.cuda.synchronize()
    step.check()
    res = {"rank": rank, "world": world, "shards": S, "scale": "cfg5", "ok": True,
           "keys_checked": [keys[f] for f in check]}
    worst_fwd = worst_bwd = 0.0
    for f in check:
        k = keys[f]
        inv, [(uv, uo)] = ikjts[(rank, f)]
        U, N = int(step.counts[f]), int(step.counts[len(keys) + f])
        same = (np.array_equal(step.inverse[f].cpu().numpy(), inv)
                and np.array_equal(step.uvalues[f][:N].cpu().numpy(), uv)
                and np.array_equal(step.uoffsets[f][:U].cpu().numpy(), uo))
        res["ok"] &= bool(same)
        ref = oracle.expand(oracle.pooled_lookup(np.searchsorted(ids[f], uv), uo, w0[f], "sum"), inv)
        ok, err = close(step.out[f].cpu().numpy(), ref)
        res["ok"] &= ok
        worst_fwd = max(worst_fwd, err)
        g64 = np.zeros((ids[f].size, D), np.float64)
        for r in range(world):
            rinv, [(ruv, ruo)] = ikjts[(r, f)]
            gu = oracle.pool_backward(grads[f][r], rinv, ruo.size)
            lids, gw = oracle.sparse_table_grad(gu, np.searchsorted(ids[f], ruv), ruo, "sum")
            g64[lids] += gw
        new = gather_rows(step, keys, f, ids[f], S, D, dev)
        ok, err = close(new - w0[f], -(np.float32(lr) * g64.astype(np.float32)))
        res["ok"] &= ok
        worst_bwd = max(worst_bwd, err)
    res["fwd_max_rel_err"], res["bwd_max_rel_err"] = worst_fwd, worst_bwd
    print(json.dumps(res), flush=True)
    step.close()
    dist.destroy_process_group()
    return 0 if res["ok"] else 1


def main():
    if os.environ.get("SCALE") == "cfg5":
        return main_cfg5()
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
