"""Row-sharded training step over NVLink peer memory (no host sync, one CUDA graph).

Same decomposition and results as `sharded.ShardedTrainStep` (SURVEY.md
§8(e); the reference only simulates ranks, trainer_sim.py:281-305): the batch
is data-parallel, every table is split into S row shards (id mod S) and the
(table, shard) pairs are placed on the ranks LPT-first.  What changes is the
transport: instead of host-planned NCCL all-to-alls, every rank maps every
other rank's exchange buffers (CUDA IPC over NVLink / NVSwitch) and

  recd_shard_count     per-(shard, unique row) counts of the local unique IDs
  recd_peer_exchange   all-gather of the per-pair counts + barrier + plan (device)
  recd_shard_dispatch  stores the IDs and row offsets straight into the owners'
                       lists at the planned offsets (NVLink stores); with one
                       shard per table the IDs are stored by the dedup's own
                       gather instead (recd_dedup_number / recd_dedup_copy)
  recd_pool_fwd_scatter owner: partial pooling of every source's rows, each
                       row stored straight into its source's receive buffer
                       over NVLink (pooling fused with the return all-to-all)
  recd_shard_combine   source: shard-order sum + avg, then recd_expand
  recd_grad_unique_scatter source: gradient of every unique row, stored
                       straight into the owners' receive buffers over NVLink
  recd_sparse_sgd      owner: deterministic sorted scatter-add + SGD (its
                       _prepare half -- the occurrence sort -- runs on a side
                       stream from the end of the dispatch, overlapping the rest)

Every size lives on the device, so the whole forward + backward is captured
once into a CUDA graph and replayed; exchanges are bounded-time barriers (a
lost peer sets the control block's error word instead of hanging).
Deterministic, bit-identical to `ShardedTrainStep` with the same S.
"""

from __future__ import annotations

import ctypes as C
from typing import Callable, Sequence

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .embedding import EmbeddingTable
from .sharded import place_pairs, shard_rows

__all__ = ["PeerShardedStep"]

_CTL_EPOCH, _CTL_ERR, _CTL_META = 64, 65, 128


class _RowSeg(C.Structure):
    _fields_ = [("src", C.c_void_p), ("dst", C.c_void_p), ("count_idx", C.c_int64),
                ("src_off_idx", C.c_int64), ("dst_off_idx", C.c_int64)]


class _DevArray:
    """__cuda_array_interface__ view of raw device memory (for torch.as_tensor)."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr,
                                         "data": (ptr, False), "version": 3}


class PeerShardedStep:
    """One rank's view of the peer-memory sharded step.  Same arguments as
    ShardedTrainStep; all exchange buffers are sized for the worst case at
    construction (IDs: the sum of every source's value capacity per pair)."""

    def __init__(self, keys: Sequence[str], batch_size: int, value_caps: dict[str, int],
                 table_rows: dict[str, int], dim: int,
                 make_table: Callable[[str, int, int], EmbeddingTable], op: str = "sum",
                 lr: float = 0.01, shards: int | None = None, group=None, device=None,
                 timeout_s: float = 10.0, overlap: bool = True):
        self.lib = L = _lib.load()
        self.overlap = bool(overlap)
        self.group = group
        self.R = R = dist.get_world_size(group)
        self.rank = rank = dist.get_rank(group)
        self.keys = list(keys)
        self.F = F = len(self.keys)
        self.S = S = int(shards or R)
        self.B = B = int(batch_size)
        self.D = D = int(dim)
        self.P = P = F * S
        if op == "max":
            raise ValueError("the row-sharded path supports sum/avg pooling")
        if S < 1 or P > 256 or R > 64:
            raise ValueError("need 1 <= shards, features x shards <= 256, ranks <= 64")
        if D % 4:
            raise ValueError("dim must be a multiple of 4 (16-byte rows)")
        self.op, self.mode_id, self.lr = op, _lib.POOL_MODES[op], float(lr)
        self.timeout_ns = int(timeout_s * 1e9)
        self.dev = dev = device or torch.device("cuda", torch.cuda.current_device())
        self._side = torch.cuda.Stream(dev)       # owner-side occurrence sort (overlap)
        self._ev_fork, self._ev_join = torch.cuda.Event(), torch.cuda.Event()
        i64, f32 = torch.int64, torch.float32
        self.caps = [max(int(value_caps[k]), 1) for k in self.keys]
        mine_caps = torch.tensor(self.caps, dtype=i64, device=dev)
        got = [torch.empty_like(mine_caps) for _ in range(R)]
        dist.all_gather(got, mine_caps, group=group)
        self.caps_all = np.stack([g.cpu().numpy() for g in got])          # [R, F]
        tot = self.caps_all.sum(axis=0)
        self.place = place_pairs([float(tot[p // S]) / S for p in range(P)], R)
        self.owned_by = [[p for p in range(P) if self.place[p] == r] for r in range(R)]
        self.mine = self.owned_by[rank]
        self.Q = Q = len(self.mine)
        self.capid = [int(self.caps_all[:, p // S].sum()) for p in self.mine]
        self.tables = {}
        for p in self.mine:
            k = self.keys[p // S]
            t = make_table(k, p % S, shard_rows(int(table_rows[k]), S, p % S))
            if t.dim != D:
                raise ValueError("all tables must share one embedding dim")
            self.tables[p] = t
        # symmetric exchange allocation: every rank can compute every layout
        self.layouts = [self._layout(r) for r in range(R)]
        lay = self.layouts[rank]
        ptr = C.c_void_p()
        _lib.check(L.recd_peer_alloc(lay["bytes"], C.byref(ptr)), "recd_peer_alloc")
        self._own = ptr.value
        h = (C.c_uint8 * 64)()
        _lib.check(L.recd_peer_export(self._own, h), "recd_peer_export")
        ht = torch.tensor(list(bytes(h)), dtype=torch.uint8, device=dev)
        hs = [torch.empty_like(ht) for _ in range(R)]
        dist.all_gather(hs, ht, group=group)
        self.bases, self._imported = [], []
        for r in range(R):
            if r == rank:
                self.bases.append(self._own)
                continue
            buf = (C.c_uint8 * 64).from_buffer_copy(bytes(hs[r].cpu().tolist()))
            out = C.c_void_p()
            _lib.check(L.recd_peer_import(buf, C.byref(out)), "recd_peer_import")
            self.bases.append(out.value)
            self._imported.append(out.value)
        W = 2 * P
        self.i_plan = _CTL_META + R * W
        self.i_own_counts = self.i_plan + 2 * P
        self.i_own_base = self.i_own_counts + 2 * Q
        nctl = int(L.recd_peer_ctl_words(R, P, Q))
        self.ctl_ptr = self._own + lay["ctl"]
        self.ctl = torch.as_tensor(_DevArray(self.ctl_ptr, nctl, "<i8"), device=dev)
        # local KJT + IKJT
        self.in_values = [torch.zeros(c, dtype=i64, device=dev) for c in self.caps]
        self.in_offsets = [torch.zeros(B, dtype=i64, device=dev) for _ in self.keys]
        self.nvalues = list(self.caps)
        self.inverse = [torch.empty(B, dtype=i64, device=dev) for _ in self.keys]
        self.uoffsets = [torch.empty(B, dtype=i64, device=dev) for _ in self.keys]
        self.uvalues = [torch.empty(c, dtype=i64, device=dev) for c in self.caps]
        self.counts = torch.zeros(2 * F, dtype=i64, device=dev)
        self.rowoff = [torch.empty(S * B, dtype=i64, device=dev) for _ in self.keys]
        self.totals = torch.zeros(P, dtype=i64, device=dev)
        self.part_out = [torch.empty((R * B, D), dtype=f32, device=dev) for _ in self.mine]
        self.gradG = torch.empty((F * B, D), dtype=f32, device=dev)
        self.pooled = [torch.empty((B, D), dtype=f32, device=dev) for _ in self.keys]
        self.out = [torch.empty((B, D), dtype=f32, device=dev) for _ in self.keys]
        self.grad_out = [torch.empty((B, D), dtype=f32, device=dev) for _ in self.keys]
        self.err = torch.full((2,), _lib.RECD_NO_ERROR, dtype=i64, device=dev)
        self.s_dedup = torch.empty(max(L.recd_dedup_scratch_bytes(F, F, B), 256),
                                   dtype=torch.uint8, device=dev)
        self.s_count = torch.empty(max(L.recd_shard_count_scratch_bytes(F, S, B), 256),
                                   dtype=torch.uint8, device=dev)
        self.s_grad = torch.empty(max(L.recd_grad_unique_scratch_bytes(F, B), 256),
                                  dtype=torch.uint8, device=dev)
        self.s_sgd = torch.empty(max(L.recd_sparse_sgd_scratch_bytes(max(Q, 1),
                                                                     _lib.i64s(self.capid or [1])),
                                     256), dtype=torch.uint8, device=dev)
        self._pointers()
        self.graph = None
        self.trace = False
        self.marks: list = []
        torch.cuda.synchronize(dev)
        dist.barrier(group=group)   # every control block is zeroed before any exchange

    # ------------------------------------------------------------ layout
    def _layout(self, r: int) -> dict:
        R, S, B, D, P = self.R, self.S, self.B, self.D, self.P
        owned = self.owned_by[r]
        off = 0

        def take(nbytes: int) -> int:
            nonlocal off
            o = off
            off += (int(nbytes) + 255) // 256 * 256
            return o

        lay = {"ctl": take(8 * self.lib.recd_peer_ctl_words(R, P, len(owned))),
               "part": take(4 * P * B * D)}                      # partial rows received (source)
        for q, p in enumerate(owned):
            lay[("ids", q)] = take(8 * int(self.caps_all[:, p // S].sum()))
            lay[("ro", q)] = take(8 * R * B)
            lay[("grad", q)] = take(4 * R * B * D)
        lay["bytes"] = off
        return lay

    def _peer(self, r: int, what, q: int | None = None) -> int:
        key = what if q is None else (what, q)
        return self.bases[r] + self.layouts[r][key]

    def _pointers(self):
        R, S, B, D, F, P, Q, rank = self.R, self.S, self.B, self.D, self.F, self.P, self.Q, self.rank
        Pp, I = _lib.ptrs, _lib.i64s
        W = 2 * P
        self.a_gsizes = _lib.i32s([1] * F)
        self.a_in_values, self.a_in_offsets = Pp(self.in_values), Pp(self.in_offsets)
        self.a_nvalues = I(self.nvalues)
        self.a_inverse, self.a_uoffsets = Pp(self.inverse), Pp(self.uoffsets)
        self.a_uvalues, self.a_rowoff = Pp(self.uvalues), Pp(self.rowoff)
        self.a_peer_ctl = Pp([self._peer(r, "ctl") for r in range(R)])
        self.a_owned = _lib.i32s(self.mine)
        dst_ids, dst_ro = [], []
        for p in range(P):
            o = self.place[p]
            qo = self.owned_by[o].index(p)
            dst_ids.append(self._peer(o, "ids", qo))
            dst_ro.append(self._peer(o, "ro", qo))
        self.a_dst_ids, self.a_dst_ro = Pp(dst_ids), Pp(dst_ro)
        self.a_no_ids = Pp([0] * P)                                 # dispatch: row offsets only
        self.a_id_base = Pp([self.ctl_ptr + 8 * (self.i_plan + p) for p in range(P)])
        self.plan_ptr = self.ctl_ptr + 8 * self.i_plan
        self.own_counts_ptr = self.ctl_ptr + 8 * self.i_own_counts
        self.a_tables = Pp([self.tables[p].weights for p in self.mine])
        self.a_rows = I([self.tables[p].rows for p in self.mine])
        self.a_own_ids = Pp([self._peer(rank, "ids", q) for q in range(Q)])
        self.a_own_ro = Pp([self._peer(rank, "ro", q) for q in range(Q)])
        self.a_own_grad = Pp([self._peer(rank, "grad", q) for q in range(Q)])
        self.a_part_out = Pp(self.part_out)
        self.a_capid = I(self.capid or [1])
        row = 4 * D
        self.a_blocks = Pp([self._peer(rank, "part") + p * B * row for p in range(P)])
        self.a_pooled, self.a_out = Pp(self.pooled), Pp(self.out)
        self.a_grad_out = Pp(self.grad_out)
        self.a_gradG = Pp([self.gradG.data_ptr() + f * B * row for f in range(F)])
        # owner -> sources: rows [owner_row_base[q][s], + U_s) of part_out[q]
        segs = []
        for q, p in enumerate(self.mine):
            for s in range(R):
                segs.append((self.part_out[q].data_ptr(), self._peer(s, "part") + p * B * row,
                             _CTL_META + s * W + P + p, self.i_own_base + q * R + s, -1))
        self.part_segs = self._segs(segs)
        # fused return: owned pair q's rows of source s start at own_base[q][s]
        # (device, exchange plan) and go to source s's receive buffer of pair p
        self.a_seg_row0 = Pp([self.ctl_ptr + 8 * (self.i_own_base + q * R) for q in range(Q)] or [0])
        self.a_seg_dst = Pp([self._peer(s2, "part") + p * B * row for p in self.mine for s2 in range(R)]
                            or [0])
        # source -> owners: all U rows of feature f(p) at src_row_base[p]
        segs = []
        for p in range(P):
            o = self.place[p]
            segs.append((self.gradG.data_ptr() + (p // S) * B * row,
                         self._peer(o, "grad", self.owned_by[o].index(p)),
                         _CTL_META + rank * W + P + p, -1, self.i_plan + P + p))
        self.grad_segs = self._segs(segs)
        # fused push: feature f's rows go to the owner of each pair (f, j) at that
        # owner's row base for this rank (device, exchange plan)
        self.a_gseg_dst = Pp([self._peer(self.place[p], "grad", self.owned_by[self.place[p]].index(p))
                              for p in range(P)])
        self.a_gseg_row0 = Pp([self.ctl_ptr + 8 * (self.i_plan + P + p) for p in range(P)])

    def _segs(self, segs) -> tuple[torch.Tensor, int]:
        arr = (_RowSeg * max(len(segs), 1))()
        for i, (src, dst, ci, so, do) in enumerate(segs):
            arr[i] = _RowSeg(src, dst, ci, so, do)
        host = torch.frombuffer(bytearray(bytes(arr)), dtype=torch.uint8)
        return host.to(self.dev), len(segs)

    def close(self):
        """Unmap the peers' buffers and free this rank's exchange allocation."""
        if getattr(self, "_own", None):
            torch.cuda.synchronize(self.dev)
            dist.barrier(group=self.group)
            for ptr in self._imported:
                self.lib.recd_peer_close(ptr)
            self._imported = []
            dist.barrier(group=self.group)
            self.ctl = None
            self.lib.recd_peer_free(self._own)
            self._own = None

    # ------------------------------------------------------------- inputs
    def load_batch(self, values, offsets):
        for f, k in enumerate(self.keys):
            v = torch.as_tensor(values[k])
            n = v.numel()
            if n > self.caps[f]:
                raise ValueError(f"feature {k!r}: batch exceeds the step's capacity")
            if self.graph is not None and n != self.nvalues[f]:
                raise ValueError("the captured graph is bound to the value counts it was "
                                 "captured with; capture() again")
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
    def _mark(self, name: str):
        if self.trace:
            e = torch.cuda.Event(enable_timing=True)
            e.record(torch.cuda.current_stream(self.dev))
            self.marks.append((name, e))

    def phase_ms(self) -> dict:
        torch.cuda.synchronize(self.dev)
        out = {}
        for (_, e0), (n1, e1) in zip(self.marks, self.marks[1:]):
            out[n1] = out.get(n1, 0.0) + e0.elapsed_time(e1)
        return out

    def _exchange(self, s, with_counts: bool):
        rc = self.lib.recd_peer_exchange(self.R, self.rank, self.P, self.S, self.Q, self.a_owned,
                                         self.a_peer_ctl,
                                         self.totals.data_ptr() if with_counts else None,
                                         self.counts.data_ptr(), self.timeout_ns, s)
        _lib.check(rc, "recd_peer_exchange")

    def forward(self):
        L, s = self.lib, _lib.stream_ptr(self.dev)
        R, S, B, D, F, Q = self.R, self.S, self.B, self.D, self.F, self.Q
        self.marks = []
        self._mark("start")
        dd = (F, self.a_gsizes, B, self.a_in_values, self.a_in_offsets, self.a_nvalues,
              self.a_inverse, self.a_uoffsets, self.a_uvalues, self.counts.data_ptr())
        fused = S == 1  # the gather of the unique values doubles as the ID dispatch
        if fused:
            rc = L.recd_dedup_number(*dd, self.s_dedup.data_ptr(), self.s_dedup.numel(), s)
            _lib.check(rc, "recd_dedup_number")
        else:
            rc = L.recd_dedup(*dd, self.s_dedup.data_ptr(), self.s_dedup.numel(), s)
            _lib.check(rc, "recd_dedup")
        self._mark("dedup")
        rc = L.recd_shard_count(F, S, B, self.a_uvalues, self.a_uoffsets, self.counts.data_ptr(),
                                self.a_rowoff, self.totals.data_ptr(), self.s_count.data_ptr(),
                                self.s_count.numel(), s)
        _lib.check(rc, "recd_shard_count")
        self._mark("shard_count")
        self._exchange(s, True)
        self._mark("exchange_counts")
        if fused:
            # unique values gathered straight into the owners' ID lists (plan bases)
            rc = L.recd_dedup_copy(*dd, self.a_dst_ids, self.a_id_base, self.s_dedup.data_ptr(),
                                   self.s_dedup.numel(), s)
            _lib.check(rc, "recd_dedup_copy")
        rc = L.recd_shard_dispatch(F, S, B, self.a_uvalues, self.a_uoffsets, self.counts.data_ptr(),
                                   self.a_rowoff, self.totals.data_ptr(), self.plan_ptr,
                                   self.plan_ptr + 8 * self.P,
                                   self.a_no_ids if fused else self.a_dst_ids, self.a_dst_ro, s)
        _lib.check(rc, "recd_shard_dispatch")
        self._exchange(s, False)
        self._mark("dispatch_ids")
        if Q and self.overlap:
            # the owner's ID lists are complete: sort the occurrences by ID on a
            # side stream while the forward, grad_unique and the push run
            main = torch.cuda.current_stream(self.dev)
            self._ev_fork.record(main)
            self._side.wait_event(self._ev_fork)
            _lib.check(L.recd_sparse_sgd_prepare(*self._sgd_args(self._side.cuda_stream)),
                       "recd_sparse_sgd_prepare")
            self._ev_join.record(self._side)
        if Q:
            # owner pooling fused with the return all-to-all: every partial row
            # is stored straight into its source's receive buffer over NVLink
            rc = L.recd_pool_fwd_scatter(Q, R * B, D, _lib.POOL_MODES["sum"], self.a_tables,
                                         self.a_rows, self.a_own_ids, self.a_own_ro,
                                         self.own_counts_ptr, R, self.a_seg_row0, self.a_seg_dst,
                                         self.err.data_ptr(), s)
            _lib.check(rc, "recd_pool_fwd_scatter(owner)")
        self._mark("owner_pool")
        self._exchange(s, False)
        self._mark("return_partials")
        if S == 1 and self.mode_id == _lib.POOL_MODES["sum"]:
            # one shard per table: the owner's partial row IS the pooled row
            rc = L.recd_expand(F, B, D, self.a_inverse, self.a_blocks, self.a_out, s)
        else:
            rc = L.recd_shard_combine(F, S, B, D, self.mode_id, self.a_blocks, self.a_uoffsets,
                                      self.counts.data_ptr(), self.a_pooled, s)
            _lib.check(rc, "recd_shard_combine")
            rc = L.recd_expand(F, B, D, self.a_inverse, self.a_pooled, self.a_out, s)
        _lib.check(rc, "recd_expand")
        self._mark("combine_expand")

    def backward(self):
        L, s = self.lib, _lib.stream_ptr(self.dev)
        R, B, D, F, Q = self.R, self.B, self.D, self.F, self.Q
        if self.S <= 8:
            # segment reduce fused with the push: every unique-row gradient is
            # stored straight into its owners' receive buffers over NVLink
            rc = L.recd_grad_unique_scatter(F, B, D, self.mode_id, self.a_uoffsets,
                                            self.counts.data_ptr(), self.a_inverse, self.a_grad_out,
                                            self.S, self.a_gseg_row0, self.a_gseg_dst,
                                            self.s_grad.data_ptr(), self.s_grad.numel(), s)
            _lib.check(rc, "recd_grad_unique_scatter")
            self._mark("grad_unique")
        else:
            rc = L.recd_grad_unique(F, B, D, self.mode_id, self.a_uoffsets, self.counts.data_ptr(),
                                    self.a_inverse, self.a_grad_out, self.a_gradG,
                                    self.s_grad.data_ptr(), self.s_grad.numel(), s)
            _lib.check(rc, "recd_grad_unique")
            self._mark("grad_unique")
            segs, n = self.grad_segs
            _lib.check(L.recd_peer_copy_rows(n, segs.data_ptr(), self.ctl_ptr, 4 * D, B, s),
                       "recd_peer_copy_rows")
        self._exchange(s, False)
        self._mark("push_grads")
        if Q and self.overlap:
            torch.cuda.current_stream(self.dev).wait_event(self._ev_join)
            _lib.check(L.recd_sparse_sgd_finish(*self._sgd_args(s)), "recd_sparse_sgd_finish")
        elif Q:
            _lib.check(L.recd_sparse_sgd(*self._sgd_args(s)), "recd_sparse_sgd")
        self._mark("owner_sgd")

    def _sgd_args(self, s):
        return (self.Q, self.R * self.B, self.D, self.a_tables, self.a_rows, self.a_own_ids,
                self.a_own_ro, self.a_capid, self.own_counts_ptr, self.a_own_grad,
                C.c_float(self.lr), 1, None, None, None, self.s_sgd.data_ptr(), self.s_sgd.numel(), s)

    def run(self):
        self.forward()
        self.backward()

    def capture(self, warmup: bool = True) -> None:
        """Record run() into a CUDA graph (replay() then launches it whole)."""
        if warmup:
            self.run()
        torch.cuda.synchronize(self.dev)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.run()

    def replay(self) -> None:
        if self.graph is None:
            self.run()
        else:
            self.graph.replay()

    def check(self) -> None:
        """Raise if an exchange timed out or a lookup saw an out-of-range ID."""
        if int(self.ctl[_CTL_ERR].item()):
            raise RuntimeError("peer exchange timed out (a rank did not arrive)")
        bad = int(self.err[0].item())
        if bad != _lib.RECD_NO_ERROR:
            raise IndexError(f"owner lookup: local ID out of range (code {bad:#x})")

    def host_counts(self):
        c = self.counts.cpu().tolist()
        return c[: self.F], c[self.F:]
