"""Row-sharded multi-GPU training step of the IKJT hot path.

SURVEY.md §8(e): the batch is data-parallel (rank r owns rows
[r*B, (r+1)*B) of the global batch, deduplicated locally -- exactly
`slice_ikjt_rows` / `split_batch`, trainer_sim.py:394-446) and every embedding
table is row-sharded over the R ranks: owner(id) = id mod R, local row
id div R.  The reference only simulates ranks and shards table-wise
(trainer_sim.py:202-214, 281-305); here the exchange is real (NCCL over
NVLink) and carries only

  forward   deduplicated IDs (per owner, per unique row)   source -> owner
            partially pooled rows, one per unique row       owner  -> source
  backward  gradient rows of the unique rows                source -> owner

The inverse_lookup never travels (trainer_sim.py:268-275).  Owners pool
their share of every unique row (recd_pool_fwd over the received jagged
lists), sources add the R partials in fixed owner order (recd_shard_combine)
and expand; the backward computes grad_u at the source (recd_grad_unique) and
the owners run the deterministic sorted scatter-add + SGD on their shard
(recd_sparse_sgd).  Results are deterministic; versus one GPU the pooled sums
change fp32 association (partial sums), so parity is within the north_star
1e-5 tolerance, while IDs / inverse stay bit-exact.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .embedding import EmbeddingTable

__all__ = ["ShardedTrainStep", "ExchangePlan", "plan_exchange", "shard_rows"]


def shard_rows(rows: int, num_ranks: int, rank: int) -> int:
    """Rows of a table held by `rank` under owner(id) = id mod R."""
    return (rows - rank + num_ranks - 1) // num_ranks


@dataclass
class ExchangePlan:
    """Host-side split sizes of one step's exchanges (from the count all-to-all).

    send_ids[o][f]  IDs of feature f this rank sends to owner o
    send_rows[f]    unique rows of feature f here (sent to every owner)
    recv_ids[s][f]  IDs of feature f received from source s
    recv_rows[s][f] unique rows of feature f at source s
    """

    R: int
    F: int
    send_ids: np.ndarray
    send_rows: np.ndarray
    recv_ids: np.ndarray
    recv_rows: np.ndarray

    def send_id_base(self, f: int, o: int) -> int:
        return int(self.send_ids[:o, f].sum())

    def recv_id_base(self, f: int, s: int) -> int:
        return int(self.recv_ids[:s, f].sum())

    def recv_row_base(self, f: int, s: int) -> int:
        return int(self.recv_rows[:s, f].sum())

    def owner_rows(self, f: int) -> int:
        return int(self.recv_rows[:, f].sum())

    def owner_ids(self, f: int) -> int:
        return int(self.recv_ids[:, f].sum())


def plan_exchange(send_meta: np.ndarray, recv_meta: np.ndarray) -> ExchangePlan:
    """send_meta / recv_meta: [R, 2F] int64 rows exchanged by the count
    all-to-all: [o, f] = IDs of f for owner o, [o, F + f] = rows of f."""
    R, two_f = send_meta.shape
    F = two_f // 2
    return ExchangePlan(R, F, send_meta[:, :F].copy(), send_meta[0, F:].copy(),
                        recv_meta[:, :F].copy(), recv_meta[:, F:].copy())


class ShardedTrainStep:
    """One rank's view of the row-sharded step (all buffers preallocated at
    worst case; host syncs only for the exchange split sizes)."""

    def __init__(self, keys: Sequence[str], batch_size: int, value_caps: dict[str, int],
                 local_tables: dict[str, EmbeddingTable], op: str = "sum", lr: float = 0.01,
                 group=None, device=None):
        self.lib = _lib.load()
        self.group = group
        self.R = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.keys = list(keys)
        self.F = len(self.keys)
        self.B = int(batch_size)
        self.op = op
        self.mode_id = _lib.POOL_MODES[op]
        self.lr = float(lr)
        self.dev = device or torch.device("cuda", torch.cuda.current_device())
        self.tables = [local_tables[k] for k in self.keys]
        self.D = self.tables[0].dim
        R, B, D, F, dev = self.R, self.B, self.D, self.F, self.dev
        i64, f32 = torch.int64, torch.float32
        self.caps = [max(int(value_caps[k]), 1) for k in self.keys]
        # local KJT + IKJT
        self.in_values = [torch.zeros(c, dtype=i64, device=dev) for c in self.caps]
        self.in_offsets = [torch.zeros(B, dtype=i64, device=dev) for _ in self.keys]
        self.nvalues = list(self.caps)
        self.inverse = [torch.empty(B, dtype=i64, device=dev) for _ in self.keys]
        self.uoffsets = [torch.empty(B, dtype=i64, device=dev) for _ in self.keys]
        self.uvalues = [torch.empty(c, dtype=i64, device=dev) for c in self.caps]
        self.counts = torch.zeros(2 * F, dtype=i64, device=dev)
        # bucketize (send side)
        self.ids_send = [torch.empty(c, dtype=i64, device=dev) for c in self.caps]
        self.rowcnt_send = [torch.empty(R * B, dtype=i64, device=dev) for _ in self.keys]
        self.totals = torch.zeros(F * R, dtype=i64, device=dev)
        # owner side (worst case: every source sends everything)
        self.ocaps = [R * c for c in self.caps]
        self.ids_recv = [torch.empty(c, dtype=i64, device=dev) for c in self.ocaps]
        self.rc_recv = [torch.zeros(R * B, dtype=i64, device=dev) for _ in self.keys]
        self.ro = [torch.zeros(R * B, dtype=i64, device=dev) for _ in self.keys]
        self.part = [torch.empty((R * B, D), dtype=f32, device=dev) for _ in self.keys]
        self.grad_recv = [torch.empty((R * B, D), dtype=f32, device=dev) for _ in self.keys]
        self.counts_owner = torch.zeros(2 * F, dtype=i64, device=dev)
        # packed exchange buffers: one NCCL collective per direction
        #   A  (int64) per peer: [row counts of f = 0..F-1][IDs of f = 0..F-1]
        #   B  (fp32)  per peer: partially pooled rows of f = 0..F-1
        #   G  (fp32)  this rank's unique-row gradients of f = 0..F-1 (all-gathered)
        capA = R * (F * B + sum(self.caps))
        self.sendA = torch.empty(capA, dtype=i64, device=dev)
        self.recvA = torch.empty(capA, dtype=i64, device=dev)
        self.sendB = torch.empty((R * F * B, D), dtype=f32, device=dev)
        self.recvB = torch.empty((R * F * B, D), dtype=f32, device=dev)
        self.gradG = torch.empty((F * B, D), dtype=f32, device=dev)
        self.recvG = torch.empty((R * F * B, D), dtype=f32, device=dev)
        # source side outputs
        self.pooled = [torch.empty((B, D), dtype=f32, device=dev) for _ in self.keys]
        self.out = [torch.empty((B, D), dtype=f32, device=dev) for _ in self.keys]
        self.grad_out = [torch.empty((B, D), dtype=f32, device=dev) for _ in self.keys]
        self.err = torch.empty(2, dtype=i64, device=dev)  # [first bad ID, work counter]
        self.meta_send = torch.zeros((R, 2 * F), dtype=i64, device=dev)
        self.meta_recv = torch.zeros((R, 2 * F), dtype=i64, device=dev)
        # batched-copy descriptor staging (one pinned host + device table per call site)
        nseg = 2 * R * F
        db = self.lib.recd_batched_copy_desc_bytes(nseg)
        self.cp_host = [torch.empty(db, dtype=torch.uint8).pin_memory() for _ in range(4)]
        self.cp_dev = [torch.empty(db, dtype=torch.uint8, device=dev) for _ in range(4)]
        L = self.lib
        self.s_dedup = torch.empty(max(L.recd_dedup_scratch_bytes(F, F, B), 256), dtype=torch.uint8,
                                   device=dev)
        self.s_shard = torch.empty(max(L.recd_shard_scratch_bytes(F, R, B), 256), dtype=torch.uint8,
                                   device=dev)
        self.s_grad = torch.empty(max(L.recd_grad_unique_scratch_bytes(F, B), 256), dtype=torch.uint8,
                                  device=dev)
        self.s_sgd = torch.empty(max(L.recd_sparse_sgd_scratch_bytes(F, _lib.i64s(self.ocaps)), 256),
                                 dtype=torch.uint8, device=dev)
        self.s_scan = torch.empty(
            max(L.recd_exclusive_scan_scratch_bytes(F, _lib.i64s([R * B] * F)), 256),
            dtype=torch.uint8, device=dev)
        self._args()
        self.plan: ExchangePlan | None = None
        self.trace = False           # record CUDA events between sub-phases
        self.marks: list = []

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

    def _args(self):
        P, I = _lib.ptrs, _lib.i64s
        self.a_gsizes = _lib.i32s([1] * self.F)
        self.a_in_values, self.a_in_offsets = P(self.in_values), P(self.in_offsets)
        self.a_nvalues = I(self.nvalues)
        self.a_inverse, self.a_uoffsets, self.a_uvalues = P(self.inverse), P(self.uoffsets), P(self.uvalues)
        self.a_ids_send, self.a_rowcnt = P(self.ids_send), P(self.rowcnt_send)
        self.a_tables = P([t.weights for t in self.tables])
        self.a_rows = I([t.rows for t in self.tables])
        self.a_ids_recv, self.a_ro, self.a_rc = P(self.ids_recv), P(self.ro), P(self.rc_recv)
        self.a_part = P(self.part)
        self.a_pooled, self.a_out = P(self.pooled), P(self.out)
        self.a_grad_out, self.a_grad_recv = P(self.grad_out), P(self.grad_recv)
        self.a_ocaps = I(self.ocaps)

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

    # --------------------------------------------------------- exchanges
    def _copy(self, site: int, segs):
        """segs: [(src_ptr, dst_ptr, bytes)] -> one batched-copy launch."""
        if not segs:
            return
        rc = self.lib.recd_batched_copy(len(segs), _lib.ptrs([x[0] for x in segs]),
                                        _lib.ptrs([x[1] for x in segs]),
                                        _lib.i64s([x[2] for x in segs]),
                                        self.cp_host[site].data_ptr(), self.cp_dev[site].data_ptr(),
                                        _lib.stream_ptr(self.dev))
        _lib.check(rc, "recd_batched_copy")

    def _exchange_counts(self) -> ExchangePlan:
        R, F = self.R, self.F
        tot = self.totals.view(F, R)  # [f, o]
        self.meta_send[:, :F].copy_(tot.t())
        self.meta_send[:, F:].copy_(self.counts[:F].unsqueeze(0).expand(R, F))
        dist.all_to_all_single(self.meta_recv, self.meta_send, group=self.group)
        host = torch.stack([self.meta_send, self.meta_recv]).cpu().numpy()
        return plan_exchange(host[0], host[1])

    # ---------------------------------------------------------------- step
    def forward(self):
        L, s = self.lib, _lib.stream_ptr(self.dev)
        R, B, D, F = self.R, self.B, self.D, self.F
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
        # 2. IDs per owner
        rc = L.recd_shard_bucketize(F, R, B, self.a_uvalues, self.a_uoffsets, self.counts.data_ptr(),
                                    self.a_ids_send, self.a_rowcnt, self.totals.data_ptr(),
                                    self.s_shard.data_ptr(), self.s_shard.numel(), s)
        _lib.check(rc, "recd_shard_bucketize")
        self._mark("bucketize")
        # 3. split sizes (the one host sync of the step)
        pl = self.plan = self._exchange_counts()
        # 4. IDs + per-row counts to the owners: pack [o][counts f..][IDs f..],
        #    one all-to-all, unpack per feature in source order
        U = [int(x) for x in pl.send_rows]
        segs, send_split, pos = [], [], 0
        for o in range(R):
            start = pos
            for f in range(F):
                segs.append((self.rowcnt_send[f].data_ptr() + 8 * o * B,
                             self.sendA.data_ptr() + 8 * pos, 8 * U[f]))
                pos += U[f]
            for f in range(F):
                n = int(pl.send_ids[o, f])
                segs.append((self.ids_send[f].data_ptr() + 8 * pl.send_id_base(f, o),
                             self.sendA.data_ptr() + 8 * pos, 8 * n))
                pos += n
            send_split.append(pos - start)
        self._copy(0, segs)
        recv_split = [int(pl.recv_rows[src].sum() + pl.recv_ids[src].sum()) for src in range(R)]
        dist.all_to_all_single(self.recvA[:sum(recv_split)], self.sendA[:pos], recv_split,
                               send_split, group=self.group)
        segs, pos = [], 0
        for src in range(R):
            for f in range(F):
                n = int(pl.recv_rows[src, f])
                segs.append((self.recvA.data_ptr() + 8 * pos,
                             self.rc_recv[f].data_ptr() + 8 * pl.recv_row_base(f, src), 8 * n))
                pos += n
            for f in range(F):
                n = int(pl.recv_ids[src, f])
                segs.append((self.recvA.data_ptr() + 8 * pos,
                             self.ids_recv[f].data_ptr() + 8 * pl.recv_id_base(f, src), 8 * n))
                pos += n
        self._copy(1, segs)
        self._mark("exchange_ids")
        # 5. owner: row offsets of the received jagged lists, owner counts
        orows = [pl.owner_rows(f) for f in range(F)]
        oids = [pl.owner_ids(f) for f in range(F)]
        self.counts_owner.copy_(torch.tensor(orows + oids, dtype=torch.int64))
        rc = L.recd_exclusive_scan(F, self.a_rc, self.a_ro, _lib.i64s([max(n, 1) for n in orows]),
                                   None, None, self.s_scan.data_ptr(), self.s_scan.numel(), s)
        _lib.check(rc, "recd_exclusive_scan")
        # 6. owner: partial pooled rows (sum of the owned share of every row)
        rc = L.recd_pool_fwd(F, R * B, D, _lib.POOL_MODES["sum"],
                             self.a_tables, self.a_rows, self.a_ids_recv, self.a_ro,
                             self.counts_owner.data_ptr(), None, self.a_part, None,
                             self.err.data_ptr(), s)
        _lib.check(rc, "recd_pool_fwd(owner)")
        self._mark("owner_pool")
        # 7. partial rows back to the sources: pack [s][f rows], one all-to-all;
        #    the source receives [o][f][U_f rows] and sums the owners in order
        row = 4 * D
        segs, send_split, pos = [], [], 0
        for src in range(R):
            start = pos
            for f in range(F):
                n = int(pl.recv_rows[src, f])
                segs.append((self.part[f].data_ptr() + row * pl.recv_row_base(f, src),
                             self.sendB.data_ptr() + row * pos, row * n))
                pos += n
            send_split.append((pos - start) * D)
        self._copy(2, segs)
        tot_u = sum(U)
        dist.all_to_all_single(self.recvB.view(-1)[:R * tot_u * D], self.sendB.view(-1)[:pos * D],
                               [tot_u * D] * R, send_split, group=self.group)
        self._mark("exchange_pooled")
        # 8. source: owner-order sum (+ avg scaling), expansion.  Feature f of
        #    owner o starts at row o * tot_u + sum(U[:f]) of recvB.
        ret = [self.recvB[sum(U[:f]):] for f in range(F)]
        rc = L.recd_shard_combine(F, R, max(tot_u, 1), D, self.mode_id, _lib.ptrs(ret),
                                  self.a_uoffsets, self.counts.data_ptr(), self.a_pooled, s)
        _lib.check(rc, "recd_shard_combine")
        rc = L.recd_expand(F, B, D, self.a_inverse, self.a_pooled, self.a_out, s)
        _lib.check(rc, "recd_expand")
        self._mark("combine_expand")

    def backward(self):
        L, s = self.lib, _lib.stream_ptr(self.dev)
        R, B, D, F = self.R, self.B, self.D, self.F
        pl = self.plan
        U = [int(x) for x in pl.send_rows]
        # grad_u of every feature written packed: feature f at row sum(U[:f])
        gptr = [self.gradG[sum(U[:f]):] for f in range(F)]
        rc = L.recd_grad_unique(F, B, D, self.mode_id, self.a_uoffsets, self.counts.data_ptr(),
                                self.a_inverse, self.a_grad_out, _lib.ptrs(gptr),
                                self.s_grad.data_ptr(), self.s_grad.numel(), s)
        _lib.check(rc, "recd_grad_unique")
        self._mark("grad_unique")
        # every owner needs every source's unique-row grads: one all-gather
        # (padded to the largest source), then unpack per feature in source order
        rows_of = pl.recv_rows.sum(axis=1).astype(np.int64)  # per source
        mx = int(rows_of.max())
        dist.all_gather_into_tensor(self.recvG.view(-1)[:R * mx * D], self.gradG.view(-1)[:mx * D],
                                    group=self.group)
        row = 4 * D
        segs = []
        for src in range(R):
            pos = src * mx
            for f in range(F):
                n = int(pl.recv_rows[src, f])
                segs.append((self.recvG.data_ptr() + row * pos,
                             self.grad_recv[f].data_ptr() + row * pl.recv_row_base(f, src), row * n))
                pos += n
        self._copy(3, segs)
        self._mark("exchange_grads")
        rc = L.recd_sparse_sgd(F, R * B, D, self.a_tables, self.a_rows, self.a_ids_recv, self.a_ro,
                               self.a_ocaps, self.counts_owner.data_ptr(), self.a_grad_recv,
                               C.c_float(self.lr), 1, None, None, None, self.s_sgd.data_ptr(),
                               self.s_sgd.numel(), s)
        _lib.check(rc, "recd_sparse_sgd")
        self._mark("owner_sgd")

    def run(self):
        self.forward()
        self.backward()

    def host_counts(self):
        c = self.counts.cpu().tolist()
        return c[: self.F], c[self.F:]
