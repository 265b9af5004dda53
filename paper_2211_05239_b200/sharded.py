"""Row-sharded multi-GPU training step of the IKJT hot path.

SURVEY.md §8(e): the batch is data-parallel (rank r owns rows [r*B, (r+1)*B)
of the global batch and deduplicates them locally -- exactly `slice_ikjt_rows`
/ `split_batch`, trainer_sim.py:394-446) and every embedding table is
row-sharded: shard j of table f holds the IDs with id mod S == j (local row
id div S).  The F*S (table, shard) pairs are placed on the R ranks
longest-processing-time first, so S trades exchange volume (S partial rows per
unique row) against load balance; S = R with one shard per rank is plain
row-wise sharding.  The reference only simulates ranks and shards table-wise
(trainer_sim.py:202-214, 281-305); here the exchange is real (NCCL over
NVLink) and carries only

  forward   deduplicated IDs (per shard, per unique row)    source -> owner
            partially pooled rows, one per (unique row, shard) owner -> source
  backward  gradient rows of the unique rows                 source -> owners

The inverse_lookup never travels (trainer_sim.py:268-275).  Owners pool their
share of every unique row (recd_pool_fwd over the received jagged lists),
sources add the S partials in fixed shard order (recd_shard_combine) and
expand; the backward computes grad_u at the source (recd_grad_unique) and the
owners run the deterministic sorted scatter-add + SGD on their shards
(recd_sparse_sgd).  Partial-row and gradient exchanges are issued per feature
group as async NCCL all-to-alls, overlapping the next group's owner compute.
Exchange buffers are sized exactly from the step's count exchange (grow-only).
Results are deterministic; versus one GPU the pooled sums change fp32
association (partial sums), so parity is within the north_star 1e-5
tolerance, while IDs / inverse stay bit-exact.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Callable, Sequence

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .embedding import EmbeddingTable

__all__ = ["ShardedTrainStep", "ExchangePlan", "plan_exchange", "shard_rows", "place_pairs",
           "auto_shards"]


def shard_rows(rows: int, num_shards: int, shard: int) -> int:
    """Rows of table shard `shard` under shard(id) = id mod S (local row id div S)."""
    return (rows - shard + num_shards - 1) // num_shards


def place_pairs(weights: Sequence[float], num_ranks: int) -> list[int]:
    """Longest-processing-time placement of (table, shard) pairs on ranks.
    Deterministic (ties: lower pair index first, then lower rank), so every
    rank computes the same placement from the same weights."""
    order = sorted(range(len(weights)), key=lambda p: (-weights[p], p))
    load = [0.0] * num_ranks
    place = [0] * len(weights)
    for p in order:
        r = min(range(num_ranks), key=lambda q: (load[q], q))
        place[p] = r
        load[r] += weights[p]
    return place


def auto_shards(weights: Sequence[float], table_bytes: Sequence[int], num_ranks: int,
                budget_bytes: float) -> int:
    """Smallest S whose LPT placement keeps every rank's table shards within
    budget_bytes.  Fewer shards = fewer partial rows per unique row (the
    exchange and owner work grow with S), so S > 1 only when tables must be
    split to fit HBM (or to balance a few very hot tables)."""
    F = len(weights)
    for S in range(1, num_ranks + 1):
        place = place_pairs([weights[p // S] / S for p in range(F * S)], num_ranks)
        load = [0.0] * num_ranks
        for p, r in enumerate(place):
            load[r] += table_bytes[p // S] / S
        if max(load) <= budget_bytes:
            return S
    raise ValueError("tables do not fit the HBM budget even fully row-sharded")


@dataclass
class ExchangePlan:
    """Host-side split sizes of one step's exchanges (from the count all-to-all).

    Pairs p = f * S + j.  send_ids[p] / send_rows[p]: IDs / unique rows this
    rank sends for pair p (to its owner); recv_ids[s, p] / recv_rows[s, p]:
    what source s sends this rank for pair p (0 for pairs owned elsewhere)."""

    R: int
    P: int
    send_ids: np.ndarray
    send_rows: np.ndarray
    recv_ids: np.ndarray
    recv_rows: np.ndarray

    def owner_rows(self, p: int) -> int:
        return int(self.recv_rows[:, p].sum())

    def owner_ids(self, p: int) -> int:
        return int(self.recv_ids[:, p].sum())

    def recv_row_base(self, p: int, s: int) -> int:
        return int(self.recv_rows[:s, p].sum())

    def recv_id_base(self, p: int, s: int) -> int:
        return int(self.recv_ids[:s, p].sum())


def plan_exchange(send_meta: np.ndarray, recv_meta: np.ndarray) -> ExchangePlan:
    """send_meta / recv_meta: [R, 2P] int64 rows exchanged by the count
    all-to-all: [d, p] = IDs of pair p for rank d, [d, P + p] = its rows
    (zero unless d owns p)."""
    R, two_p = send_meta.shape
    P = two_p // 2
    return ExchangePlan(R, P, send_meta[:, :P].sum(axis=0), send_meta[:, P:].sum(axis=0),
                        recv_meta[:, :P].copy(), recv_meta[:, P:].copy())


class ShardedTrainStep:
    """One rank's view of the sharded step.  `make_table(key, shard, rows)`
    returns the EmbeddingTable of a (table, shard) pair placed on this rank;
    `table_rows[key]` is the full table's row count."""

    def __init__(self, keys: Sequence[str], batch_size: int, value_caps: dict[str, int],
                 table_rows: dict[str, int], dim: int,
                 make_table: Callable[[str, int, int], EmbeddingTable], op: str = "sum",
                 lr: float = 0.01, shards: int | None = None, group=None, device=None,
                 ngroups: int = 4):
        self.lib = L = _lib.load()
        self.group = group
        self.R = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.keys = list(keys)
        self.F = len(self.keys)
        self.S = int(shards or self.R)
        self.B = int(batch_size)
        self.D = int(dim)
        self.op = op
        self.mode_id = _lib.POOL_MODES[op]
        self.lr = float(lr)
        self.dev = device or torch.device("cuda", torch.cuda.current_device())
        R, S, B, D, F, dev = self.R, self.S, self.B, self.D, self.F, self.dev
        if not 1 <= S or F * S > 256:
            raise ValueError("need 1 <= shards and features x shards <= 256")
        i64, f32 = torch.int64, torch.float32
        self.caps = [max(int(value_caps[k]), 1) for k in self.keys]
        # identical placement on every rank: weights from the global value counts
        tot = torch.tensor(self.caps, dtype=torch.float64, device=dev)
        dist.all_reduce(tot, group=group)
        tot = tot.cpu().tolist()
        self.place = place_pairs([tot[p // S] / S for p in range(F * S)], R)
        self.mine = [p for p in range(F * S) if self.place[p] == self.rank]
        if len(self.mine) > 64:
            raise ValueError("more than 64 (table, shard) pairs on one rank")
        self.by_dest = [[p for p in range(F * S) if self.place[p] == d] for d in range(R)]
        self.tables = {}
        for p in self.mine:
            k = self.keys[p // S]
            t = make_table(k, p % S, shard_rows(int(table_rows[k]), S, p % S))
            if t.dim != D:
                raise ValueError("all tables must share one embedding dim")
            self.tables[p] = t
        # local KJT + IKJT
        self.in_values = [torch.zeros(c, dtype=i64, device=dev) for c in self.caps]
        self.in_offsets = [torch.zeros(B, dtype=i64, device=dev) for _ in self.keys]
        self.nvalues = list(self.caps)
        self.inverse = [torch.empty(B, dtype=i64, device=dev) for _ in self.keys]
        self.uoffsets = [torch.empty(B, dtype=i64, device=dev) for _ in self.keys]
        self.uvalues = [torch.empty(c, dtype=i64, device=dev) for c in self.caps]
        self.counts = torch.zeros(2 * F, dtype=i64, device=dev)
        # IDs bucketized by shard (send side)
        self.ids_send = [torch.empty(c, dtype=i64, device=dev) for c in self.caps]
        self.rowcnt_send = [torch.empty(S * B, dtype=i64, device=dev) for _ in self.keys]
        self.totals = torch.zeros(F * S, dtype=i64, device=dev)  # [f * S + j]
        # source outputs
        self.pooled = [torch.empty((B, D), dtype=f32, device=dev) for _ in self.keys]
        self.out = [torch.empty((B, D), dtype=f32, device=dev) for _ in self.keys]
        self.grad_out = [torch.empty((B, D), dtype=f32, device=dev) for _ in self.keys]
        self.gradG = torch.empty((F * B, D), dtype=f32, device=dev)
        self.err = torch.empty(2, dtype=i64, device=dev)  # [first bad ID, work counter]
        place = torch.tensor(self.place, dtype=i64, device=dev)
        self.pmask = (place[None, :] == torch.arange(R, device=dev)[:, None]).to(i64)  # [R, P]
        self.pair_feature = torch.arange(F, device=dev).repeat_interleave(S)      # f(p)
        self.meta_send = torch.zeros((R, 2 * F * S), dtype=i64, device=dev)
        self.meta_recv = torch.zeros((R, 2 * F * S), dtype=i64, device=dev)
        self.s_dedup = torch.empty(max(L.recd_dedup_scratch_bytes(F, F, B), 256),
                                   dtype=torch.uint8, device=dev)
        self.s_shard = torch.empty(max(L.recd_shard_scratch_bytes(F, S, B), 256),
                                   dtype=torch.uint8, device=dev)
        self.s_grad = torch.empty(max(L.recd_grad_unique_scratch_bytes(F, B), 256),
                                  dtype=torch.uint8, device=dev)
        self._bufs: dict = {}
        P = _lib.ptrs
        self.a_gsizes = _lib.i32s([1] * F)
        self.a_in_values, self.a_in_offsets = P(self.in_values), P(self.in_offsets)
        self.a_nvalues = _lib.i64s(self.nvalues)
        self.a_inverse, self.a_uoffsets, self.a_uvalues = P(self.inverse), P(self.uoffsets), P(self.uvalues)
        self.a_ids_send, self.a_rowcnt = P(self.ids_send), P(self.rowcnt_send)
        self.a_grad_out = P(self.grad_out)
        # contiguous feature groups: the exchange of group g overlaps the owner
        # compute of group g + 1
        ng = max(1, min(ngroups, F))
        bounds = [round(i * F / ng) for i in range(ng + 1)]
        self.groups = [list(range(bounds[i], bounds[i + 1])) for i in range(ng)
                       if bounds[i + 1] > bounds[i]]
        self.g_idx = [torch.tensor(g + [F + f for f in g], dtype=i64, device=dev)
                      for g in self.groups]
        self.g_counts = [torch.zeros(2 * len(g), dtype=i64, device=dev) for g in self.groups]
        self.g_mine = [[p for p in self.mine if p // S in g] for g in self.groups]
        # batched-copy descriptor staging: one pinned host + device table per call site
        # (0: pack IDs, 1: unpack IDs, then per group: pack partials, pack grads, unpack grads)
        nsite = 2 + 3 * len(self.groups)
        db = L.recd_batched_copy_desc_bytes(2 * R * F * S + 8)
        self.cp_host = [torch.empty(db, dtype=torch.uint8).pin_memory() for _ in range(nsite)]
        self.cp_dev = [torch.empty(db, dtype=torch.uint8, device=dev) for _ in range(nsite)]
        self.plan: ExchangePlan | None = None
        self.trace = False           # record CUDA events between sub-phases
        self.marks: list = []

    # -------------------------------------------------------------- utils
    def _buf(self, name: str, n: int, dtype=torch.int64, cols: int = 0) -> torch.Tensor:
        """Grow-only device buffer of at least max(n, 1) rows."""
        n = max(int(n), 1)
        b = self._bufs.get(name)
        if b is None or b.shape[0] < n:
            shape = (n + n // 4 + 1, cols) if cols else (n + n // 4 + 1,)
            b = torch.empty(shape, dtype=dtype, device=self.dev)
            self._bufs[name] = b
        return b

    def _mark(self, name: str):
        if self.trace:
            e = torch.cuda.Event(enable_timing=True)
            e.record(torch.cuda.current_stream(self.dev))
            self.marks.append((name, e))

    def phase_ms(self) -> dict:
        """Durations between consecutive marks of the last traced step."""
        torch.cuda.synchronize(self.dev)
        out = {}
        for (n0, e0), (n1, e1) in zip(self.marks, self.marks[1:]):
            out[n1] = out.get(n1, 0.0) + e0.elapsed_time(e1)
        return out

    def _copy(self, site: int, segs):
        """segs: [(src_ptr, dst_ptr, bytes)] -> one batched-copy launch."""
        segs = [x for x in segs if x[2] > 0]
        if not segs:
            return
        rc = self.lib.recd_batched_copy(len(segs), _lib.ptrs([x[0] for x in segs]),
                                        _lib.ptrs([x[1] for x in segs]),
                                        _lib.i64s([x[2] for x in segs]),
                                        self.cp_host[site].data_ptr(), self.cp_dev[site].data_ptr(),
                                        _lib.stream_ptr(self.dev))
        _lib.check(rc, "recd_batched_copy")

    # ------------------------------------------------------------- inputs
    def load_batch(self, values, offsets):
        for f, k in enumerate(self.keys):
            v = torch.as_tensor(values[k])
            n = v.numel()
            if n > self.caps[f]:
                raise ValueError(f"feature {k!r}: batch exceeds the step's capacity")
            self.in_values[f][:n].copy_(v)
            self.in_offsets[f].copy_(torch.as_tensor(offsets[k]))
            self.nvalues[f] = n
        self.a_nvalues = _lib.i64s(self.nvalues)

    def fill_grad_out(self, seed: int = 1):
        g = torch.Generator(device=self.dev)
        g.manual_seed(seed)
        for t in self.grad_out:
            t.normal_(generator=g)

    # ---------------------------------------------------------------- step
    def _exchange_counts(self) -> ExchangePlan:
        P = self.F * self.S
        rows = self.counts[self.pair_feature]  # U_f(p)
        torch.mul(self.pmask, self.totals[None, :], out=self.meta_send[:, :P])
        torch.mul(self.pmask, rows[None, :], out=self.meta_send[:, P:])
        dist.all_to_all_single(self.meta_recv, self.meta_send, group=self.group)
        host = torch.stack([self.meta_send, self.meta_recv]).cpu().numpy()
        return plan_exchange(host[0], host[1])

    def forward(self):
        L, s = self.lib, _lib.stream_ptr(self.dev)
        R, S, B, D, F = self.R, self.S, self.B, self.D, self.F
        if self.op == "max":
            raise ValueError("the row-sharded path supports sum/avg pooling")
        self.marks = []
        self._mark("start")
        # 1. local dedup
        rc = L.recd_dedup(F, self.a_gsizes, B, self.a_in_values, self.a_in_offsets, self.a_nvalues,
                          self.a_inverse, self.a_uoffsets, self.a_uvalues, self.counts.data_ptr(),
                          self.s_dedup.data_ptr(), self.s_dedup.numel(), s)
        _lib.check(rc, "recd_dedup")
        self._mark("dedup")
        # 2. unique IDs bucketized by shard: ids_send[f] = [shard 0][shard 1]..
        rc = L.recd_shard_bucketize(F, S, B, self.a_uvalues, self.a_uoffsets, self.counts.data_ptr(),
                                    self.a_ids_send, self.a_rowcnt, self.totals.data_ptr(),
                                    self.s_shard.data_ptr(), self.s_shard.numel(), s)
        _lib.check(rc, "recd_shard_bucketize")
        self._mark("bucketize")
        # 3. split sizes (the one host sync of the step)
        pl = self.plan = self._exchange_counts()
        mine, by_dest = self.mine, self.by_dest
        sid = [int(x) for x in pl.send_ids]
        U = [int(pl.send_rows[f * S]) for f in range(F)]
        ibase = [0] * (F * S)
        for f in range(F):
            for j in range(1, S):
                ibase[f * S + j] = ibase[f * S + j - 1] + sid[f * S + j - 1]
        # 4. IDs + per-row counts to the owners, packed per destination as
        #    [row counts of its pairs][IDs of its pairs]; one all-to-all
        sendA = self._buf("sendA", sum(U[p // S] + sid[p] for p in range(F * S)))
        segs, send_split, pos = [], [], 0
        for d in range(R):
            start = pos
            for p in by_dest[d]:
                f, j = divmod(p, S)
                segs.append((self.rowcnt_send[f].data_ptr() + 8 * j * B,
                             sendA.data_ptr() + 8 * pos, 8 * U[f]))
                pos += U[f]
            for p in by_dest[d]:
                segs.append((self.ids_send[p // S].data_ptr() + 8 * ibase[p],
                             sendA.data_ptr() + 8 * pos, 8 * sid[p]))
                pos += sid[p]
            send_split.append(pos - start)
        self._copy(0, segs)
        recv_split = [int(pl.recv_rows[src].sum() + pl.recv_ids[src].sum()) for src in range(R)]
        recvA = self._buf("recvA", sum(recv_split))
        dist.all_to_all_single(recvA[:sum(recv_split)], sendA[:pos], recv_split, send_split,
                               group=self.group)
        # owner side, exact sizes: unpack per pair in source order
        self.orows = {p: pl.owner_rows(p) for p in mine}
        self.oids = {p: pl.owner_ids(p) for p in mine}
        rc_recv = {p: self._buf(f"rc{p}", self.orows[p]) for p in mine}
        self.ro = {p: self._buf(f"ro{p}", self.orows[p]) for p in mine}
        self.ids_recv = {p: self._buf(f"ids{p}", self.oids[p]) for p in mine}
        segs, pos = [], 0
        for src in range(R):
            for p in mine:
                n = int(pl.recv_rows[src, p])
                segs.append((recvA.data_ptr() + 8 * pos,
                             rc_recv[p].data_ptr() + 8 * pl.recv_row_base(p, src), 8 * n))
                pos += n
            for p in mine:
                n = int(pl.recv_ids[src, p])
                segs.append((recvA.data_ptr() + 8 * pos,
                             self.ids_recv[p].data_ptr() + 8 * pl.recv_id_base(p, src), 8 * n))
                pos += n
        self._copy(1, segs)
        self._mark("exchange_ids")
        # 5. owner: row offsets of the received jagged lists, owner counts
        if mine:
            cap = [max(self.orows[p], 1) for p in mine]
            scr = self._buf("scan", L.recd_exclusive_scan_scratch_bytes(len(mine), _lib.i64s(cap)),
                            torch.uint8)
            rc = L.recd_exclusive_scan(len(mine), _lib.ptrs([rc_recv[p] for p in mine]),
                                       _lib.ptrs([self.ro[p] for p in mine]), _lib.i64s(cap),
                                       None, None, scr.data_ptr(), scr.numel(), s)
            _lib.check(rc, "recd_exclusive_scan")
        host = [self.orows[p] for gp in self.g_mine for p in gp] + \
               [self.oids[p] for gp in self.g_mine for p in gp]
        oc = torch.tensor(host or [0], dtype=torch.int64).to(self.dev)
        self.counts_owner, n_m, o0 = [], len(host) // 2, 0
        for gi, gp in enumerate(self.g_mine):
            self.counts_owner.append(torch.cat([oc[o0:o0 + len(gp)], oc[n_m + o0:n_m + o0 + len(gp)]]))
            o0 += len(gp)
            torch.index_select(self.counts, 0, self.g_idx[gi], out=self.g_counts[gi])
        self._mark("owner_scan")
        # 6-7. per feature group: owner partial pooling, packed partial rows back
        #      to the sources (async all-to-all on NCCL's stream overlaps the
        #      next group's pooling)
        row = 4 * D
        works = []
        for gi, g in enumerate(self.groups):
            gp = self.g_mine[gi]
            part = {p: self._buf(f"part{p}", self.orows[p], torch.float32, D) for p in gp}
            if gp:
                rc = L.recd_pool_fwd(len(gp), R * B, D, _lib.POOL_MODES["sum"],
                                     _lib.ptrs([self.tables[p].weights for p in gp]),
                                     _lib.i64s([self.tables[p].rows for p in gp]),
                                     _lib.ptrs([self.ids_recv[p] for p in gp]),
                                     _lib.ptrs([self.ro[p] for p in gp]),
                                     self.counts_owner[gi].data_ptr(), None,
                                     _lib.ptrs([part[p] for p in gp]), None,
                                     self.err.data_ptr(), s)
                _lib.check(rc, "recd_pool_fwd(owner)")
            sendB = self._buf(f"sendB{gi}", sum(self.orows[p] for p in gp), torch.float32, D)
            segs, send_split, pos = [], [], 0
            for src in range(R):
                start = pos
                for p in gp:
                    n = int(pl.recv_rows[src, p])
                    segs.append((part[p].data_ptr() + row * pl.recv_row_base(p, src),
                                 sendB.data_ptr() + row * pos, row * n))
                    pos += n
                send_split.append((pos - start) * D)
            self._copy(2 + gi, segs)
            # from owner o: the pairs of this group it owns, U_f rows each
            recv_split, blocks, rpos = [], {}, 0
            for o in range(R):
                start = rpos
                for p in by_dest[o]:
                    if p // S in g:
                        blocks[p] = rpos
                        rpos += U[p // S]
                recv_split.append((rpos - start) * D)
            recvB = self._buf(f"recvB{gi}", rpos, torch.float32, D)
            work = dist.all_to_all_single(recvB.view(-1)[:rpos * D], sendB.view(-1)[:pos * D],
                                          recv_split, send_split, group=self.group, async_op=True)
            works.append((work, recvB, blocks))
        self._mark("owner_pool")
        # 8. per group: shard-order sum (+ avg scaling), expansion
        for gi, g in enumerate(self.groups):
            work, recvB, blocks = works[gi]
            work.wait()
            blk = [recvB[blocks[f * S + j]:] for f in g for j in range(S)]
            rc = L.recd_shard_combine(len(g), S, B, D, self.mode_id, _lib.ptrs(blk),
                                      _lib.ptrs([self.uoffsets[f] for f in g]),
                                      self.g_counts[gi].data_ptr(),
                                      _lib.ptrs([self.pooled[f] for f in g]), s)
            _lib.check(rc, "recd_shard_combine")
            rc = L.recd_expand(len(g), B, D, _lib.ptrs([self.inverse[f] for f in g]),
                               _lib.ptrs([self.pooled[f] for f in g]),
                               _lib.ptrs([self.out[f] for f in g]), s)
            _lib.check(rc, "recd_expand")
        self._U = U
        self._mark("exchange_combine")

    def backward(self):
        L, s = self.lib, _lib.stream_ptr(self.dev)
        R, S, B, D, F = self.R, self.S, self.B, self.D, self.F
        pl, U, by_dest = self.plan, self._U, self.by_dest
        gbase = np.concatenate([[0], np.cumsum(U)]).astype(np.int64).tolist()
        rc = L.recd_grad_unique(F, B, D, self.mode_id, self.a_uoffsets, self.counts.data_ptr(),
                                self.a_inverse, self.a_grad_out,
                                _lib.ptrs([self.gradG[gbase[f]:] for f in range(F)]),
                                self.s_grad.data_ptr(), self.s_grad.numel(), s)
        _lib.check(rc, "recd_grad_unique")
        self._mark("grad_unique")
        # per group, to every owner of one of its pairs: that feature's
        # unique-row gradients; all issued now so they run back to back while
        # the owners scatter the earlier groups
        row, ng = 4 * D, len(self.groups)
        works = []
        for gi, g in enumerate(self.groups):
            n_send = sum(U[p // S] for d in range(R) for p in by_dest[d] if p // S in g)
            sendG = self._buf(f"sendG{gi}", n_send, torch.float32, D)
            segs, send_split, pos = [], [], 0
            for d in range(R):
                start = pos
                for p in by_dest[d]:
                    f = p // S
                    if f in g:
                        segs.append((self.gradG.data_ptr() + row * gbase[f],
                                     sendG.data_ptr() + row * pos, row * U[f]))
                        pos += U[f]
                send_split.append((pos - start) * D)
            self._copy(2 + ng + gi, segs)
            gp = self.g_mine[gi]
            recv_split = [sum(int(pl.recv_rows[src, p]) for p in gp) * D for src in range(R)]
            nrecv = sum(recv_split) // D
            recvG = self._buf(f"recvG{gi}", nrecv, torch.float32, D)
            work = dist.all_to_all_single(recvG.view(-1)[:nrecv * D], sendG.view(-1)[:pos * D],
                                          recv_split, send_split, group=self.group, async_op=True)
            works.append((work, recvG))
        for gi, g in enumerate(self.groups):
            work, recvG = works[gi]
            work.wait()
            gp = self.g_mine[gi]
            if not gp:
                continue
            # received [source][pair][row]; each pair's SGD wants [source][row]
            grad = {p: self._buf(f"grad{p}", self.orows[p], torch.float32, D) for p in gp}
            segs, pos = [], 0
            for src in range(R):
                for p in gp:
                    n = int(pl.recv_rows[src, p])
                    segs.append((recvG.data_ptr() + row * pos,
                                 grad[p].data_ptr() + row * pl.recv_row_base(p, src), row * n))
                    pos += n
            self._copy(2 + 2 * ng + gi, segs)
            caps = [max(self.oids[p], 1) for p in gp]
            scr = self._buf("sgd", L.recd_sparse_sgd_scratch_bytes(len(gp), _lib.i64s(caps)),
                            torch.uint8)
            rc = L.recd_sparse_sgd(len(gp), R * B, D,
                                   _lib.ptrs([self.tables[p].weights for p in gp]),
                                   _lib.i64s([self.tables[p].rows for p in gp]),
                                   _lib.ptrs([self.ids_recv[p] for p in gp]),
                                   _lib.ptrs([self.ro[p] for p in gp]), _lib.i64s(caps),
                                   self.counts_owner[gi].data_ptr(),
                                   _lib.ptrs([grad[p] for p in gp]), C.c_float(self.lr), 1,
                                   None, None, None, scr.data_ptr(), scr.numel(), s)
            _lib.check(rc, "recd_sparse_sgd")
        self._mark("exchange_sgd")

    def run(self):
        self.forward()
        self.backward()

    def host_counts(self):
        c = self.counts.cpu().tolist()
        return c[: self.F], c[self.F:]
