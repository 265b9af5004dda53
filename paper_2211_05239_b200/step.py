"""One training step of the IKJT hot path over preallocated device buffers.

`TrainStep` owns every buffer a step touches (KJT input slots, IKJT outputs
at worst-case size, pooled/expanded outputs, gradients, scratch) and the
ctypes argument arrays, so a step is four C-ABI calls with no allocation and
no host synchronisation -- capturable as one CUDA graph:

    recd_dedup_ex    KJT -> IKJT for every group              (skipped in "kjt" mode)
    recd_pool_fwd    pooled lookup over unique rows
    recd_expand      expansion of the pooled rows to [B, D] via inverse_lookup
    recd_pool_bwd    grad segment-reduce + sorted scatter-add + fused SGD

With overlap=True (default) the backward is split: recd_pool_bwd_prepare
(inverse CSR + occurrence sort, gradient-independent) runs on a side stream
right after the dedup, concurrently with the pooled lookup and expansion,
and recd_pool_bwd_finish joins on the main stream.

pipeline=True goes one step further, the way the reference splits its reader
from its trainer (reader.convert builds the IKJTs of the next batch while
the trainer runs, reader.py:160-175): the IKJT-only half of batch i+1 -- the
dedup and the backward's prepare half -- runs on the side stream while the
main stream runs batch i's pooled lookup, expansion and backward + SGD.
Nothing of batch i+1 touches the tables, so every batch's results are
bit-identical to the sequential step; two IKJT stages alternate (stage =
slot = step parity) and each parity is one captured CUDA graph.

This is the device-side equivalent of one `forward_iteration`'s sparse part
(trainer_sim.py:484-574) plus the backward the reference does not have.
Like the reference's iteration, a step may mix deduplicated groups with
plain KJT keys (`plain=`, trainer_sim.py:562-574): the plain keys skip the
dedup, are pooled per batch row and take the backward's identity path, in
the same calls (and graph) as the deduplicated features.
"""

from __future__ import annotations

import ctypes as C
import os
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


class _Stage:
    """One set of IKJT outputs + the scratch of the dedup and the backward
    (the prepare half writes the backward scratch, the finish half reads it)."""

    def __init__(self, step: "TrainStep"):
        dev, B, F, i64 = step.dev, step.B, step.F, torch.int64
        lib = step.lib
        Fd = step.Fd
        self.inverse = [torch.empty(B, dtype=i64, device=dev) for _ in step.groups]
        self.uoffsets = [torch.empty(B, dtype=i64, device=dev) for _ in step.keys[:Fd]]
        self.uvalues = [torch.empty(c, dtype=i64, device=dev) for c in step.caps[:Fd]]
        # counts of the step's features [U per feature, N_u per feature]; with
        # plain keys the dedup writes its own [2 Fd] (dc_sub) and the plain
        # keys' entries are B and the slot's value counts
        self.dcounts = torch.zeros(2 * F, dtype=i64, device=dev)
        self.dcounts[Fd:F] = B
        self.dc_sub = torch.zeros(2 * Fd, dtype=i64, device=dev) if Fd < F else self.dcounts
        self.err = torch.full((2,), _lib.RECD_NO_ERROR, dtype=i64, device=dev)
        self.dedup_scratch = torch.empty(
            max(lib.recd_dedup_scratch_bytes(max(len(step.groups), 1), max(Fd, 1), B), 256),
            dtype=torch.uint8, device=dev)
        self.bwd_scratch = torch.empty(
            max(lib.recd_pool_bwd_scratch_bytes(F, B, step.D, _lib.i64s(step.caps)), 256),
            dtype=torch.uint8, device=dev)


class _Args:
    """ctypes argument arrays of one (stage, input slot) pair."""

    def __init__(self, step: "TrainStep", stage: int, slot: int):
        L, st = _lib, step.stages[stage]
        vals, offs = step.slot_values[slot], step.slot_offsets[slot]
        self.gsizes = L.i32s([len(g) for g in step.groups])
        self.in_values, self.in_offsets = L.ptrs(vals), L.ptrs(offs)
        self.in_counts_ptr = step.in_counts[slot, step.F:].data_ptr()
        self.inverse_g = L.ptrs(st.inverse)
        self.uoffsets, self.uvalues = L.ptrs(st.uoffsets), L.ptrs(st.uvalues)
        self.tables = L.ptrs([t.weights for t in step.tables])
        self.rows = L.i64s([t.rows for t in step.tables])
        self.caps = L.i64s(step.caps)
        self.grad, self.out = L.ptrs(step.grad_out), L.ptrs(step.out)
        if step.mode == "dedup":
            Fd = step.Fd
            inv_f = []
            for gi, g in enumerate(step.groups):
                inv_f += [st.inverse[gi]] * len(g)
            # plain keys (after the deduplicated ones): identity inverse, the
            # KJT rows themselves, pooled straight into the batch rows
            self.inverse_f = L.ptrs(inv_f + [None] * (step.F - Fd))
            self.pooled = L.ptrs(step.pooled[:Fd] + step.out[Fd:])
            self.feat_vals_t = list(st.uvalues) + list(vals[Fd:])
            self.feat_vals = L.ptrs(self.feat_vals_t)
            self.feat_offs = L.ptrs(list(st.uoffsets) + list(offs[Fd:]))
            self.counts_ptr = st.dcounts.data_ptr()
            self.dc_out = st.dc_sub.data_ptr()
        else:
            self.inverse_f = L.ptrs([None] * step.F)
            self.pooled = self.out  # no expansion: pooled rows are the batch rows
            self.feat_vals, self.feat_offs, self.feat_vals_t = self.in_values, self.in_offsets, vals
            self.counts_ptr = step.in_counts[slot].data_ptr()


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
                 slots: int = 1, pipeline: bool = False, plain: Sequence[str] = ()):
        if mode not in ("dedup", "kjt"):
            raise ValueError(f"unknown mode {mode!r}")
        plain = tuple(plain)
        if set(plain) & {k for g in groups for k in g}:
            raise ValueError("a key is both in a dedup group and plain")
        if plain and mode != "dedup":
            raise ValueError("plain keys are for dedup mode (kjt mode has no dedup at all)")
        if op not in ("sum", "avg", "mean"):
            raise ValueError(f"the training step needs sum/avg pooling (max has no backward), got {op!r}")
        self.lib = _lib.load()
        self.groups = [tuple(g) for g in groups]
        self.plain = plain
        self.keys = [k for g in self.groups for k in g] + list(plain)
        self.F = len(self.keys)
        self.Fd = self.F - len(plain)  # deduplicated features come first
        self.B = int(batch_size)
        self.mode = mode
        self.op = op
        self.mode_id = _lib.POOL_MODES[op]
        self.lr = float(lr)
        self.overlap = bool(overlap)
        # dedup mode, big batches: the lookup writes the batch rows itself
        # through the backward's inverse CSR instead of a separate k_expand
        # (cfg2 4.53-4.57 vs 4.56-4.58 ms; cfg1 0.163 vs 0.157 ms, so not for
        # small batches).  RECD_FUSED_EXPAND=0/1 forces it off / on.
        fx = os.environ.get("RECD_FUSED_EXPAND")
        self.fused_expand = mode == "dedup" and (fx != "0" if fx else self.B >= 32768)
        self.pipeline = bool(pipeline)
        self.dev = device or torch.device("cuda", torch.cuda.current_device())
        self.tables = [tables[k] for k in self.keys]
        self.D = self.tables[0].dim
        dev, B, D, F = self.dev, self.B, self.D, self.F
        i64 = torch.int64
        self.caps = [max(int(value_caps[k]), 1) for k in self.keys]
        # KJT input slots: values, offsets, value counts (device)
        self.nslots = 2 if self.pipeline else max(1, int(slots))
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
        self.pooled = [torch.empty((B, D), dtype=torch.float32, device=dev) for _ in self.keys]
        self.out = [torch.empty((B, D), dtype=torch.float32, device=dev) for _ in self.keys]
        self.grad_out = [torch.empty((B, D), dtype=torch.float32, device=dev) for _ in self.keys]
        # IKJT stages (two alternate in pipeline mode)
        self.stages = [_Stage(self) for _ in range(2 if self.pipeline else 1)]
        self.stage = 0
        self._args: dict = {}
        self.graphs: list = [None] * self.nslots
        # RECD_SIDE_PRIORITY (e.g. -1): the side stream's occurrence sort gets
        # free SM slots ahead of the main stream's lookup
        self._side = torch.cuda.Stream(dev, priority=int(os.environ.get("RECD_SIDE_PRIORITY", "0")))
        self._ev_fork = torch.cuda.Event()
        self._ev_join = torch.cuda.Event()
        self._ev_inv = torch.cuda.Event()
        # small batches: the occurrence sort on a stream of its own, beside the
        # inverse CSR (RECD_BWD_SETUP first) -- both are latency-bound chains
        # there (cfg1 0.111 vs 0.117 ms); on big ones starting the sort early
        # only competes with the CSR and the lookup (cfg2 4.40 vs 4.24-4.28 ms).
        # RECD_SPLIT_PREP=0/1 forces it off / on.
        sp = os.environ.get("RECD_SPLIT_PREP")
        self.split_prep = (sp != "0") if sp else not self.fused_expand
        self._side2 = torch.cuda.Stream(dev) if self.split_prep else None

    # ------------------------------------------- current stage / slot views
    def _st(self, stage=None) -> _Stage:
        return self.stages[self.stage if stage is None else stage]

    def args(self, stage=None, slot=None) -> _Args:
        key = (self.stage if stage is None else stage, self.slot if slot is None else slot)
        a = self._args.get(key)
        if a is None:
            a = self._args[key] = _Args(self, *key)
        return a

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
    def inverse(self):
        return self._st().inverse

    @property
    def uoffsets(self):
        return self._st().uoffsets

    @property
    def uvalues(self):
        return self._st().uvalues

    @property
    def err(self):
        return self._st().err

    @property
    def counts(self):
        """Device int64[2F] (U per feature, N_u per feature) of the step's IKJT
        (kjt mode: B and the slot's value counts)."""
        return self._st().dcounts if self.mode == "dedup" else self.in_counts[self.slot]

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

    def use_slot(self, slot: int, stage: int | None = None) -> None:
        """Make `slot` (and `stage`) the step's current input / IKJT."""
        if not 0 <= slot < self.nslots:
            raise ValueError(f"slot {slot} out of range for {self.nslots} slots")
        self.slot = int(slot)
        if stage is not None:
            self.stage = int(stage)

    def fill_grad_out(self, seed: int = 1) -> None:
        g = torch.Generator(device=self.dev)
        g.manual_seed(seed)
        for t in self.grad_out:
            t.normal_(generator=g)

    # ---------------------------------------------------------------- step
    def dedup(self, stream: int, stage=None, slot=None) -> None:
        if self.mode != "dedup":
            return
        a, st = self.args(stage, slot), self._st(stage)
        Fd, F = self.Fd, self.F
        if Fd:
            rc = self.lib.recd_dedup_ex(len(self.groups), a.gsizes, self.B, a.in_values, a.in_offsets,
                                        a.caps, a.in_counts_ptr, 3, a.inverse_g, a.uoffsets,
                                        a.uvalues, a.dc_out, None, None,
                                        st.dedup_scratch.data_ptr(), st.dedup_scratch.numel(), stream)
            _lib.check(rc, "recd_dedup_ex")
        if Fd < F:  # assemble [U, N_u] of all features (plain keys: B, their value counts)
            s = torch.cuda.ExternalStream(stream, device=self.dev)
            with torch.cuda.stream(s):
                if Fd:
                    st.dcounts[:Fd].copy_(st.dc_sub[:Fd], non_blocking=True)
                    st.dcounts[F:F + Fd].copy_(st.dc_sub[Fd:], non_blocking=True)
                st.dcounts[F + Fd:].copy_(self.in_counts[self.slot if slot is None else slot, F + Fd:],
                                          non_blocking=True)

    def forward(self, stream: int, stage=None, slot=None, share: bool = False) -> None:
        """Pooled lookup over the unique rows (k_pool_fwd only).  share: the
        side stream's backward prepare runs beside it (RECD_POOL_SHARE)."""
        a, st = self.args(stage, slot), self._st(stage)
        mode = self.mode_id | (_lib.POOL_SHARE if share else 0)
        rc = self.lib.recd_pool_fwd(self.F, self.B, self.D, mode, a.tables, a.rows,
                                    a.feat_vals, a.feat_offs, a.counts_ptr, a.inverse_f, a.pooled,
                                    None, st.err.data_ptr(), stream)
        _lib.check(rc, "recd_pool_fwd")

    def _csr(self, stage=None, slot=None):
        """(csr_start, csr_rows) pointer arrays of the inverse CSR in the
        stage's backward scratch (recd_pool_bwd_csr; dedup mode)."""
        a = self.args(stage, slot)
        if getattr(a, "csr", None) is None:
            cs, cr = (C.c_void_p * self.F)(), (C.c_void_p * self.F)()
            args = self._bwd_args(0, stage, slot)[:-1]
            _lib.check(self.lib.recd_pool_bwd_csr(*args, cs, cr), "recd_pool_bwd_csr")
            a.csr = (cs, cr)
        return a.csr

    def forward_expand(self, stream: int, stage=None, slot=None, share: bool = False) -> None:
        """Pooled lookup with the expansion fused through the backward's inverse
        CSR (recd_pool_fwd_csr: no pooled buffer; needs BWD_INVERSE first)."""
        a, st = self.args(stage, slot), self._st(stage)
        cs, cr = self._csr(stage, slot)
        mode = self.mode_id | (_lib.POOL_SHARE if share else 0)
        rc = self.lib.recd_pool_fwd_csr(self.F, self.B, self.D, mode, a.tables, a.rows, a.feat_vals,
                                        a.feat_offs, a.counts_ptr, cs, cr, None, a.out,
                                        st.err.data_ptr(), stream)
        _lib.check(rc, "recd_pool_fwd_csr")

    def expand(self, stream: int, stage=None, slot=None) -> None:
        """out[i] = pooled[inverse[i]] (k_expand; nothing to do in kjt mode or
        for plain keys, whose lookup wrote the batch rows)."""
        if self.mode != "dedup" or self.Fd == 0:
            return
        a = self.args(stage, slot)
        rc = self.lib.recd_expand(self.Fd, self.B, self.D, a.inverse_f, a.pooled, a.out, stream)
        _lib.check(rc, "recd_expand")

    def _bwd_args(self, stream: int, stage=None, slot=None):
        a, st = self.args(stage, slot), self._st(stage)
        inv = a.inverse_f if self.mode == "dedup" else None
        return (self.F, self.B, self.D, self.mode_id, a.tables, a.rows, a.feat_vals, a.feat_offs,
                a.caps, a.counts_ptr, inv, a.grad, C.c_float(self.lr), 1, None, None, None,
                st.bwd_scratch.data_ptr(), st.bwd_scratch.numel(), stream)

    def backward(self, stream: int, stage=None, slot=None) -> None:
        _lib.check(self.lib.recd_pool_bwd(*self._bwd_args(stream, stage, slot)), "recd_pool_bwd")

    def backward_prepare(self, stream: int, stage=None, slot=None) -> None:
        """Gradient-independent half of the backward (may run on a side stream)."""
        _lib.check(self.lib.recd_pool_bwd_prepare(*self._bwd_args(stream, stage, slot)),
                   "recd_pool_bwd_prepare")

    def backward_finish(self, stream: int, stage=None, slot=None) -> None:
        _lib.check(self.lib.recd_pool_bwd_finish(*self._bwd_args(stream, stage, slot)),
                   "recd_pool_bwd_finish")

    def backward_stages(self, stages: int, stream: int, stage=None, slot=None) -> None:
        """Some of the backward's stages (_lib.BWD_*, recd_pool_bwd_stages)."""
        _lib.check(self.lib.recd_pool_bwd_stages(stages, *self._bwd_args(stream, stage, slot)),
                   "recd_pool_bwd_stages")

    def run(self, stream: int | None = None) -> None:
        """One whole step on the current slot / stage (dedup .. SGD)."""
        if stream is not None or not self.overlap:
            s = _lib.stream_ptr(self.dev) if stream is None else stream
            self.dedup(s)
            self.forward(s)
            self.expand(s)
            self.backward(s)
            return
        main = torch.cuda.current_stream(self.dev)
        if self.fused_expand:
            # main stream: dedup, inverse CSR, lookup with the expansion fused
            # through the CSR, unique-row gradients, then the scatter + SGD
            # after the side stream's occurrence sort (split_prep: the sort
            # starts right after the bookkeeping, beside the inverse CSR)
            ms = main.cuda_stream
            self.dedup(ms)
            if self.split_prep:
                self.backward_stages(_lib.BWD_SETUP, ms)
            else:
                self.backward_stages(_lib.BWD_INVERSE, ms)
            self._ev_fork.record(main)
            self._side.wait_event(self._ev_fork)
            self.backward_stages(_lib.BWD_OCCURRENCES, self._side.cuda_stream)
            self._ev_join.record(self._side)
            if self.split_prep:
                self.backward_stages(_lib.BWD_INVERSE | _lib.BWD_SETUP_DONE, ms)
            self.forward_expand(ms, share=True)
            self.backward_stages(_lib.BWD_GRAD, ms)
            main.wait_event(self._ev_join)
            self.backward_stages(_lib.BWD_SCATTER, ms)
            return
        # side stream: inverse CSR, then the occurrence sort; main stream: lookup,
        # expansion, unique-row gradients (after the CSR only, so they run while
        # the sort finishes), then the scatter + SGD after the sort
        self.dedup(main.cuda_stream)
        if self.split_prep:
            self.backward_stages(_lib.BWD_SETUP, main.cuda_stream)
        self._ev_fork.record(main)
        self._side.wait_event(self._ev_fork)
        ss = self._side.cuda_stream
        if self.split_prep:
            # inverse CSR and occurrence sort side by side on two streams
            # (latency-bound chains on small batches)
            self._side2.wait_event(self._ev_fork)
            self.backward_stages(_lib.BWD_INVERSE | _lib.BWD_SETUP_DONE, ss)
            self._ev_inv.record(self._side)
            self.backward_stages(_lib.BWD_OCCURRENCES, self._side2.cuda_stream)
            self._ev_join.record(self._side2)
        else:
            self.backward_stages(_lib.BWD_INVERSE, ss)
            self._ev_inv.record(self._side)
            self.backward_stages(_lib.BWD_OCCURRENCES, ss)
            self._ev_join.record(self._side)
        self.forward(main.cuda_stream, share=True)
        self.expand(main.cuda_stream)
        main.wait_event(self._ev_inv)
        self.backward_stages(_lib.BWD_GRAD, main.cuda_stream)
        main.wait_event(self._ev_join)
        self.backward_stages(_lib.BWD_SCATTER, main.cuda_stream)

    # ------------------------------------------------------ pipeline mode
    def prime(self, slot: int = 0) -> None:
        """Pipeline start: dedup + backward prepare of the batch in `slot` into
        stage `slot`, on the current stream."""
        s = torch.cuda.current_stream(self.dev).cuda_stream
        self.dedup(s, slot, slot)
        self.backward_prepare(s, slot, slot)

    def run_pipelined(self, p: int) -> None:
        """Step on the batch in slot p (primed into stage p) -- pooled lookup,
        expansion, backward + SGD on the main stream -- while the side stream
        deduplicates the batch in slot 1-p and prepares its backward into
        stage 1-p (the next step's IKJT)."""
        if not self.pipeline:
            raise ValueError("run_pipelined needs TrainStep(pipeline=True)")
        q = 1 - p
        main = torch.cuda.current_stream(self.dev)
        self._ev_fork.record(main)
        self._side.wait_event(self._ev_fork)
        ss = self._side.cuda_stream
        self.dedup(ss, q, q)
        self.backward_prepare(ss, q, q)
        self._ev_join.record(self._side)
        ms = main.cuda_stream
        self.forward(ms, p, p, share=True)
        self.expand(ms, p, p)
        self.backward_finish(ms, p, p)
        main.wait_event(self._ev_join)
        self.use_slot(p, p)

    def capture(self) -> None:
        """Record one CUDA graph per input slot (replay(slot) launches it):
        run() on that slot, or run_pipelined(slot) in pipeline mode.  Runs one
        eager warm-up step first (on the current slot)."""
        cur, cur_stage = self.slot, self.stage
        s = torch.cuda.Stream(self.dev)
        s.wait_stream(torch.cuda.current_stream(self.dev))
        with torch.cuda.stream(s):
            if self.pipeline:
                self.prime(cur)
                self.run_pipelined(cur)
            else:
                self.run()  # warm-up on the side stream
        torch.cuda.current_stream(self.dev).wait_stream(s)
        # the main stream's kernels (lookup, expand, backward finish) are captured
        # at high priority: when the side stream's occurrence sort runs beside
        # them, the block scheduler fills free SM slots with theirs first
        prio = int(os.environ.get("RECD_MAIN_PRIORITY", "0"))
        cap = torch.cuda.Stream(self.dev, priority=prio) if prio else None
        for k in range(self.nslots):
            self.use_slot(k, k if self.pipeline else cur_stage)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=cap):
                if self.pipeline:
                    self.run_pipelined(k)
                else:
                    self.run()
            self.graphs[k] = g
        self.use_slot(cur, cur_stage)

    def replay(self, slot: int | None = None) -> None:
        if slot is not None and slot != self.slot:
            self.use_slot(slot, slot if self.pipeline else None)
        g = self.graphs[self.slot]
        if g is None:
            if self.pipeline:
                self.run_pipelined(self.slot)
            else:
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
        vals = self.args().feat_vals_t[f]
        raise ValueError(f"feature {self.keys[f]!r}: ID {int(vals[pos])} at position {pos} "
                         f"out of range [0, {self.tables[f].rows})")

    def host_counts(self) -> StepCounts:
        c = self.counts.cpu().tolist()
        return StepCounts(c[: self.F], c[self.F:])
