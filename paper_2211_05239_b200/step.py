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
    def __init__(self, groups: Sequence[Sequence[str]], batch_size: int,
                 value_caps: dict[str, int], tables: dict[str, EmbeddingTable], op: str = "sum",
                 lr: float = 0.01, mode: str = "dedup", device=None, overlap: bool = True):
        if mode not in ("dedup", "kjt"):
            raise ValueError(f"unknown mode {mode!r}")
        self.lib = _lib.load()
        self.groups = [tuple(g) for g in groups]
        self.keys = [k for g in self.groups for k in g]
        self.F = len(self.keys)
        self.B = int(batch_size)
        self.mode = mode
        self.op = op
        self.mode_id = _lib.POOL_MODES[op]
        self.lr = float(lr)
        self.overlap = bool(overlap)
        self.dev = device or torch.device("cuda", torch.cuda.current_device())
        self.tables = [tables[k] for k in self.keys]
        self.D = self.tables[0].dim
        dev, B, D, F = self.dev, self.B, self.D, self.F
        i64 = torch.int64
        self.caps = [max(int(value_caps[k]), 1) for k in self.keys]
        # KJT input slots
        self.in_values = [torch.zeros(c, dtype=i64, device=dev) for c in self.caps]
        self.in_offsets = [torch.zeros(B, dtype=i64, device=dev) for _ in self.keys]
        self.nvalues = list(self.caps)
        # IKJT outputs (worst case) + device counts
        self.inverse = [torch.empty(B, dtype=i64, device=dev) for _ in self.groups]
        self.uoffsets = [torch.empty(B, dtype=i64, device=dev) for _ in self.keys]
        self.uvalues = [torch.empty(c, dtype=i64, device=dev) for c in self.caps]
        self.counts = torch.zeros(2 * F, dtype=i64, device=dev)
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
        self._build_args()
        self.graph = None

    # ------------------------------------------------------------- inputs
    def load_batch(self, values: dict[str, np.ndarray | torch.Tensor],
                   offsets: dict[str, np.ndarray | torch.Tensor], non_blocking=False) -> None:
        """Copy one KJT batch into the input slots (host or device sources)."""
        for f, k in enumerate(self.keys):
            v = torch.as_tensor(values[k])
            o = torch.as_tensor(offsets[k])
            n = v.numel()
            if n > self.caps[f] or o.numel() != self.B:
                raise ValueError(f"feature {k!r}: batch exceeds the step's capacity")
            self.in_values[f][:n].copy_(v, non_blocking=non_blocking)
            self.in_offsets[f].copy_(o, non_blocking=non_blocking)
            self.nvalues[f] = n
        self._build_args()
        if self.mode == "kjt":
            c = [self.B] * self.F + list(self.nvalues)
            self.counts.copy_(torch.tensor(c, dtype=torch.int64))

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
        self.a_nvalues = L.i64s(self.nvalues)
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
        rc = self.lib.recd_dedup(len(self.groups), self.a_gsizes, self.B, self.a_in_values,
                                 self.a_in_offsets, self.a_nvalues, self.a_inverse_g,
                                 self.a_uoffsets, self.a_uvalues, self.counts.data_ptr(),
                                 self.dedup_scratch.data_ptr(), self.dedup_scratch.numel(), stream)
        _lib.check(rc, "recd_dedup")

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
        """Record run() into a CUDA graph (replayed by replay())."""
        s = torch.cuda.Stream(self.dev)
        s.wait_stream(torch.cuda.current_stream(self.dev))
        with torch.cuda.stream(s):
            self.run()  # warm-up on the side stream
        torch.cuda.current_stream(self.dev).wait_stream(s)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.run()

    def replay(self) -> None:
        if self.graph is None:
            self.run()
        else:
            self.graph.replay()

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
