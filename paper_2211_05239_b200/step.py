"""One training step of the IKJT hot path over preallocated device buffers.

`TrainStep` owns every buffer a step touches (KJT input slots, IKJT outputs
at worst-case size, pooled/expanded outputs, gradients, scratch) and the
ctypes argument arrays, so a step is four C-ABI calls with no allocation and
no host synchronisation -- capturable as one CUDA graph:

    recd_dedup       KJT -> IKJT for every group              (skipped in "kjt" mode)
    recd_pool_fwd    pooled lookup over unique rows
    recd_expand      expansion of the pooled rows to [B, D] via inverse_lookup
    recd_pool_bwd    grad segment-reduce + sorted scatter-add + fused SGD

With overlap=True (default) the backward is split: recd_pool_bwd_prepare
(inverse CSR + occurrence sort, gradient-independent) runs on a side stream
right after recd_dedup, concurrently with the pooled lookup and expansion,
and recd_pool_bwd_finish joins on the main stream.

This is the device-side equivalent of one `forward_iteration`'s sparse part
(trainer_sim.py:484-574) plus the backward the reference does not have.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from . import _lib
from .embedding import EmbeddingTable

__all__ = ["TrainStep", "StepCounts"]


@dataclass
class StepCounts:
    U: list[int]      # unique rows per feature
    N_u: list[int]    # unique values per feature


class TrainStep:
    """One training step over `slots` input slots (each slot: the KJT values,
    offsets and value counts of one batch, all on the device).  With slots=2 a
    copy stream fills one slot while the step runs on the other, and
    capture() records one CUDA graph per slot, so no batch is ever copied
    device-to-device and any batch up to the value capacities replays the
    same graph (the counts are read on the device, recd_dedup_ex)."""

    def __init__(self, groups: Sequence[Sequence[str]], batch_size: int,
                 value_caps: dict[str, int], tables: dict[str, EmbeddingTable], op: str = "sum",
                 lr: float = 0.01, mode: str = "dedup", device=None, overlap: bool = True,
                 slots: int = 1):
        if mode not in ("dedup", "kjt"):
            raise ValueError(f"unknown mode {mode!r}")
        self.lib = _lib.load()
        self.groups = [tuple(g) for g in groups]
        self.keys = [k for g in self.groups for k in g]
        self.F = len(self.keys)
        self.B = int(batch_size)
        self.mode = mode
        self.op = op
        if op not in ("sum", "avg", "mean"):
            raise ValueError(f"the training step needs sum/avg pooling (max has no backward), got {op!r}")
        self.mode_id = _lib.POOL_MODES[op]
        self.lr = float(lr)
        self.overlap = bool(overlap)
        self.dev = device or torch.device("cuda", torch.cuda.current_device())
        self.tables = [tables[k] for k in self.keys]
        self.D = self.tables[0].dim
        dev, B, D, F = self.dev, self.B, self.D, self.F
        i64 = torch.int64
        self.caps = [max(int(value_caps[k]), 1) for k in self.keys]
        # KJT input slots: values, offsets, value counts (device)
        self.nslots = max(1, int(slots))
        self.slot_values = [[torch.zeros(c, dtype=i64, device=dev) for c in self.caps]
                            for _ in range(self.nslots)]
        self.slot_offsets = [[torch.zeros(B, dtype=i64, device=dev) for _ in self.keys]
                             for _ in range(self.nslots)]
        # per slot: [B] * F + the value counts -- the KJT's own counts layout
        # (recd_pool_fwd / _bwd in kjt mode), and the device counts recd_dedup_ex reads
        self.in_counts = torch.zeros((self.nslots, 2 * F), dtype=i64, device=dev)
        self.in_counts[:, :F] = B
        self.slot_nvalues = [[0] * F for _ in range(self.nslots)]
        self.slot = 0
        # IKJT outputs (worst case) + device counts
        self.inverse = [torch.empty(B, dtype=i64, device=dev) for _ in self.groups]
        self.uoffsets = [torch.empty(B, dtype=i64, device=dev) for _ in self.keys]
        self.uvalues = [torch.empty(c, dtype=i64, device=dev) for c in self.caps]
        self._dcounts = torch.zeros(2 * F, dtype=i64, device=dev)
        self.pooled = [torch.empty((B, D), dtype=torch.float32, device=dev) for _ in self.keys]
        self.out = [torch.empty((B, D), dtype=torch.float32, device=dev) for _ in self.keys]
        self.grad_out = [torch.empty((B, D), dtype=torch.float32, device=dev) for _ in self.keys]
        self.err = torch.empty(2, dtype=i64, device=dev)  # [first bad ID, work counter]
        self.dedup_scratch = torch.empty(
            max(self.lib.recd_dedup_scratch_bytes(len(self.groups), F, B), 256),
            dtype=torch.uint8, device=dev)
        self.bwd_scratch = torch.empty(
            max(self.lib.recd_pool_bwd_scratch_bytes(F, B, D, _lib.i64s(self.caps)), 256),
            dtype=torch.uint8, device=dev)
        self.graphs: list = [None] * self.nslots
        self._build_args()

    # current slot's buffers (the step's inputs)
    @property
    def in_values(self):
        return self.slot_values[self.slot]

    @property
    def in_offsets(self):
        return self.slot_offsets[self.slot]

    @property
    def nvalues(self):
        return self.slot_nvalues[self.slot]

    @property
    def counts(self):
        """Device int64[2F] (U per feature, N_u per feature) of the step's IKJT
        (kjt mode: B and the slot's value counts)."""
        return self._dcounts if self.mode == "dedup" else self.in_counts[self.slot]

    @property
    def graph(self):
        return self.graphs[self.slot]

    # ------------------------------------------------------------- inputs
    def load_batch(self, values: dict[str, np.ndarray | torch.Tensor],
                   offsets: dict[str, np.ndarray | torch.Tensor], non_blocking=False,
                   slot: int | None = None) -> None:
        """Copy one KJT batch (host or device sources) into an input slot
        (default: the current one).  Any value counts up to the capacities."""
        s = self.slot if slot is None else int(slot)
        n = []
        for f, k in enumerate(self.keys):
            v = torch.as_tensor(values[k])
            o = torch.as_tensor(offsets[k])
            if v.numel() > self.caps[f] or o.numel() != self.B:
                raise ValueError(f"feature {k!r}: batch exceeds the step's capacity")
            self.slot_values[s][f][: v.numel()].copy_(v, non_blocking=non_blocking)
            self.slot_offsets[s][f].copy_(o, non_blocking=non_blocking)
            n.append(v.numel())
        self.in_counts[s, self.F:].copy_(torch.tensor(n, dtype=torch.int64),
                                          non_blocking=non_blocking)
        self.slot_nvalues[s] = n

    def use_slot(self, slot: int) -> None:
        """Make `slot` the step's input (eager calls and replay() use it)."""
        if not 0 <= slot < self.nslots:
            raise ValueError(f"slot {slot} out of range for {self.nslots} slots")
        self.slot = int(slot)
        self._build_args()

    def fill_grad_out(self, seed: int = 1) -> None:
        g = torch.Generator(device=self.dev)
        g.manual_seed(seed)
        for t in self.grad_out:
            t.normal_(generator=g)

    # ---------------------------------------------------------------- args
    def _build_args(self) -> None:
        L = _lib
        self.a_gsizes = L.i32s([len(g) for g in self.groups])
        self.a_in_values = L.ptrs(self.in_values)
        self.a_in_offsets = L.ptrs(self.in_offsets)
        self.in_counts_ptr = self.in_counts[self.slot, self.F:].data_ptr()
        self.a_inverse_g = L.ptrs(self.inverse)
        self.a_uoffsets = L.ptrs(self.uoffsets)
        self.a_uvalues = L.ptrs(self.uvalues)
        self.a_tables = L.ptrs([t.weights for t in self.tables])
        self.a_rows = L.i64s([t.rows for t in self.tables])
        self.a_caps = L.i64s(self.caps)
        self.a_grad = L.ptrs(self.grad_out)
        self.a_out = L.ptrs(self.out)
        if self.mode == "dedup":
            inv_f = []
            for gi, g in enumerate(self.groups):
                inv_f += [self.inverse[gi]] * len(g)
            self.a_inverse_f = L.ptrs(inv_f)
            self.a_pooled = L.ptrs(self.pooled)
            self.a_feat_vals, self.a_feat_offs = self.a_uvalues, self.a_uoffsets
            self.a_feat_vals_t = self.uvalues
        else:
            self.a_inverse_f = L.ptrs([None] * self.F)
            self.a_pooled = L.ptrs(self.out)  # no expansion: pooled rows are the batch rows
            self.a_feat_vals, self.a_feat_offs = self.a_in_values, self.a_in_offsets
            self.a_feat_vals_t = self.in_values

    # ---------------------------------------------------------------- step
    def dedup(self, stream: int) -> None:
        if self.mode != "dedup":
            return
        rc = self.lib.recd_dedup_ex(len(self.groups), self.a_gsizes, self.B, self.a_in_values,
                                    self.a_in_offsets, self.a_caps, self.in_counts_ptr, 3,
                                    self.a_inverse_g, self.a_uoffsets, self.a_uvalues,
                                    self.counts.data_ptr(), None, None,
                                    self.dedup_scratch.data_ptr(), self.dedup_scratch.numel(),
                                    stream)
        _lib.check(rc, "recd_dedup_ex")

    def forward(self, stream: int) -> None:
        """Pooled lookup over the unique rows (k_pool_fwd only)."""
        rc = self.lib.recd_pool_fwd(self.F, self.B, self.D, self.mode_id, self.a_tables,
                                    self.a_rows, self.a_feat_vals, self.a_feat_offs,
                                    self.counts.data_ptr(), self.a_inverse_f, self.a_pooled,
                                    None, self.err.data_ptr(), stream)
        _lib.check(rc, "recd_pool_fwd")

    def expand(self, stream: int) -> None:
        """out[i] = pooled[inverse[i]] (k_expand; nothing to do in kjt mode)."""
        if self.mode != "dedup":
            return
        rc = self.lib.recd_expand(self.F, self.B, self.D, self.a_inverse_f, self.a_pooled,
                                  self.a_out, stream)
        _lib.check(rc, "recd_expand")

    def _bwd_args(self, stream: int):
        inv = self.a_inverse_f if self.mode == "dedup" else None
        return (self.F, self.B, self.D, self.mode_id, self.a_tables, self.a_rows, self.a_feat_vals,
                self.a_feat_offs, self.a_caps, self.counts.data_ptr(), inv, self.a_grad,
                C.c_float(self.lr), 1, None, None, None, self.bwd_scratch.data_ptr(),
                self.bwd_scratch.numel(), stream)

    def backward(self, stream: int) -> None:
        _lib.check(self.lib.recd_pool_bwd(*self._bwd_args(stream)), "recd_pool_bwd")

    def backward_prepare(self, stream: int) -> None:
        """Gradient-independent half of the backward (may run on a side stream)."""
        _lib.check(self.lib.recd_pool_bwd_prepare(*self._bwd_args(stream)), "recd_pool_bwd_prepare")

    def backward_finish(self, stream: int) -> None:
        _lib.check(self.lib.recd_pool_bwd_finish(*self._bwd_args(stream)), "recd_pool_bwd_finish")

    def run(self, stream: int | None = None) -> None:
        if stream is not None or not self.overlap:
            s = _lib.stream_ptr(self.dev) if stream is None else stream
            self.dedup(s)
            self.forward(s)
            self.expand(s)
            self.backward(s)
            return
        main = torch.cuda.current_stream(self.dev)
        if not hasattr(self, "_side"):
            self._side = torch.cuda.Stream(self.dev)
            self._ev_fork = torch.cuda.Event()
            self._ev_join = torch.cuda.Event()
        self.dedup(main.cuda_stream)
        self._ev_fork.record(main)
        self._side.wait_event(self._ev_fork)
        self.backward_prepare(self._side.cuda_stream)
        self._ev_join.record(self._side)
        self.forward(main.cuda_stream)
        self.expand(main.cuda_stream)
        main.wait_event(self._ev_join)
        self.backward_finish(main.cuda_stream)

    def capture(self) -> None:
        """Record run() into one CUDA graph per input slot (replay() launches
        the current slot's).  Runs one eager warm-up step on the current slot."""
        cur = self.slot
        s = torch.cuda.Stream(self.dev)
        s.wait_stream(torch.cuda.current_stream(self.dev))
        with torch.cuda.stream(s):
            self.run()  # warm-up on the side stream
        torch.cuda.current_stream(self.dev).wait_stream(s)
        for k in range(self.nslots):
            self.use_slot(k)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self.run()
            self.graphs[k] = g
        self.use_slot(cur)

    def replay(self, slot: int | None = None) -> None:
        if slot is not None and slot != self.slot:
            self.use_slot(slot)
        g = self.graphs[self.slot]
        if g is None:
            self.run()
        else:
            g.replay()

    def check(self) -> None:
        """Raise the reference's ValueError (trainer_sim.py:312-320) if the last
        step's lookup saw an ID outside [0, rows).  The step itself never
        synchronises; the backward skips every table update of such a batch
        (k_occ flags it, k_scatter does nothing), so the tables stay intact."""
        e = int(self.err[0].item())
        if e == _lib.RECD_NO_ERROR:
            return
        f, pos = e >> 40, e & ((1 << 40) - 1)
        vals = self.a_feat_vals_t[f]
        raise ValueError(f"feature {self.keys[f]!r}: ID {int(vals[pos])} at position {pos} "
                         f"out of range [0, {self.tables[f].rows})")

    def host_counts(self) -> StepCounts:
        c = self.counts.cpu().tolist()
        return StepCounts(c[: self.F], c[self.F:])
