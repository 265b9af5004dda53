"""Double-buffered host -> device staging of KJT batches.

The KJT of a cfg2 batch is ~1 GB of int64 per GPU, so end to end the step is
bound by the PCIe copy, not by the kernels.  `H2DPipeline` copies batch i+1
from pinned host memory on a dedicated copy stream while step i runs.

With a step that owns input slots (`TrainStep(slots=2)`: one CUDA graph per
slot, value counts read on the device) the copy goes straight into the slot
the next step reads -- values, offsets and the value counts -- and nothing is
copied device-to-device: `run(slot, replay)` makes the step wait for the
slot's copy, replays that slot's graph and releases the slot to the copy
stream when the step is done with it.  Any batch up to the capacities works.

A pipelined step (`TrainStep(pipeline=True)`) deduplicates batch i+1 on its
side stream while batch i trains, so the copy of batch i+2 goes into the slot
batch i came in (`wait_ready` / `release` around each replay).

Steps without slots (the sharded steps, whose graphs are bound to one set of
input buffers and value counts) get the slot copied into their inputs by
`install(slot)` (one device-to-device copy per step).

`rowcode=True` sends each batch row-delta coded (`rowcode.py`: one code per
row plus the IDs the device cannot rebuild -- ~16x fewer bytes on session
batches); the host encodes batch i+1 (C++ threads) while step i runs, and
`recd_rowcode_decode` rebuilds the slot's values on the copy stream.
"""

from __future__ import annotations

import os

import torch

from . import _lib

__all__ = ["H2DPipeline"]


class H2DPipeline:
    def __init__(self, step, device=None, nslots: int = 2, rowcode: bool = False,
                 threads: int = 0, raw_share: float | None = None):
        self.step = step
        self.direct = getattr(step, "nslots", 1) >= nslots
        self.dev = device or step.in_values[0].device
        self.copy = torch.cuda.Stream(self.dev)
        self.n = nslots
        if self.direct:
            self.slots = [(step.slot_values[s], step.slot_offsets[s]) for s in range(nslots)]
        else:
            self.slots = [([torch.empty_like(v) for v in step.in_values],
                           [torch.empty_like(o) for o in step.in_offsets]) for _ in range(nslots)]
        F = len(step.keys)
        self._pin_counts = [torch.zeros(F, dtype=torch.int64).pin_memory() for _ in range(nslots)]
        self._pc_done = [None] * nslots   # the last H2D copy out of _pin_counts[slot]
        self.counts = [None] * nslots
        self.ready = [torch.cuda.Event() for _ in range(nslots)]
        self.free = [torch.cuda.Event() for _ in range(nslots)]
        self._freed = [False] * nslots
        self.rowcode = bool(rowcode)
        self.threads = int(threads)
        if raw_share is None:
            raw_share = float(os.environ.get("RECD_ROWCODE_RAW_SHARE", "0"))
        self.raw_share = min(max(float(raw_share), 0.0), 1.0)
        self.h2d_bytes = [0] * nslots    # bytes the last prefetch into each slot copied
        if self.rowcode:
            B = step.B
            caps = [v.numel() for v in self.slots[0][0]]
            self._capv = caps
            self._h_codes = [torch.empty((F, B), dtype=torch.uint8).pin_memory() for _ in range(nslots)]
            self._h_lits = [[torch.empty(c, dtype=torch.int64).pin_memory() for c in caps]
                            for _ in range(nslots)]
            self._d_codes = [torch.empty((F, B), dtype=torch.uint8, device=self.dev)
                             for _ in range(nslots)]
            self._d_lits = [[torch.empty(c, dtype=torch.int64, device=self.dev) for c in caps]
                            for _ in range(nslots)]
            self._d_nv = [torch.zeros(F, dtype=torch.int64, device=self.dev) for _ in range(nslots)]
            lib = _lib.load()
            self._rc_scratch = torch.empty(max(lib.recd_rowcode_scratch_bytes(F, B), 256),
                                           dtype=torch.uint8, device=self.dev)
            self._h_done = [None] * nslots   # the last H2D copy out of the slot's host staging

    def prefetch(self, slot: int, values: dict, offsets: dict) -> None:
        """Queue the H2D copy of one batch (pinned host tensors) into `slot`."""
        vals, offs = self.slots[slot]
        n = [int(values[k].shape[0]) for k in self.step.keys]
        for f, k in enumerate(self.step.keys):
            if n[f] > vals[f].numel():
                raise ValueError(f"feature {k!r}: batch exceeds the step's capacity")
        if self.rowcode:
            self._prefetch_rowcode(slot, values, offsets, n)
            return
        self.h2d_bytes[slot] = sum(8 * (n[f] + offs[f].numel()) for f in range(len(n)))
        with torch.cuda.stream(self.copy):
            if self._freed[slot]:
                self.copy.wait_event(self.free[slot])   # the step is done reading the slot
            for f, k in enumerate(self.step.keys):
                vals[f][: n[f]].copy_(values[k], non_blocking=True)
                offs[f].copy_(offsets[k], non_blocking=True)
            if self.direct:
                pc = self._pin_counts[slot]
                if self._pc_done[slot] is not None:
                    self._pc_done[slot].synchronize()   # host buffer free again
                pc.copy_(torch.tensor(n, dtype=torch.int64))
                F = len(n)
                self.step.in_counts[slot, F:].copy_(pc, non_blocking=True)
                self._pc_done[slot] = torch.cuda.Event()
                self._pc_done[slot].record(self.copy)
            self.ready[slot].record(self.copy)
        self.counts[slot] = n

    def _prefetch_rowcode(self, slot: int, values: dict, offsets: dict, n: list) -> None:
        # encoded on the calling thread with every core: on a worker thread
        # (the caller launching steps meanwhile) e2e was 11.3-11.9 vs 10.9-11.1
        # ms per cfg2 step -- the encoder is what the host is busy with.  With
        # raw_share > 0 the largest keys (that share of the IDs) go over PCIe
        # as raw int64 first, so the copy engine works while the cores encode
        from . import rowcode
        keys = self.step.keys
        F = len(keys)
        vals, offs = self.slots[slot]
        raw = self._raw_keys(n)
        coded = [f for f in range(F) if f not in raw]
        if self._h_done[slot] is not None:
            self._h_done[slot].synchronize()     # host staging free again
        pc = self._pin_counts[slot]
        if self._pc_done[slot] is not None:
            self._pc_done[slot].synchronize()
        pc.copy_(torch.tensor(n, dtype=torch.int64))
        dc, dl, dnv = self._d_codes[slot], self._d_lits[slot], self._d_nv[slot]
        with torch.cuda.stream(self.copy):
            if self._freed[slot]:
                self.copy.wait_event(self.free[slot])   # the step is done reading the slot
            for f, k in enumerate(keys):
                o = offsets[k]
                offs[f].copy_(o if isinstance(o, torch.Tensor) else torch.from_numpy(o),
                              non_blocking=True)
            for f in sorted(raw):
                v = values[keys[f]]
                vals[f][: n[f]].copy_(v if isinstance(v, torch.Tensor) else torch.from_numpy(v),
                                      non_blocking=True)
            dnv.copy_(pc, non_blocking=True)
            if self.direct:
                self.step.in_counts[slot, F:].copy_(dnv, non_blocking=True)
        hc, hl = self._h_codes[slot], self._h_lits[slot]
        lits = [0] * F
        if coded:
            got = rowcode.encode([values[keys[f]] for f in coded], [offsets[keys[f]] for f in coded],
                                 self.step.B, [hc[f] for f in coded], [hl[f] for f in coded],
                                 self.threads)
            for f, c in zip(coded, got):
                lits[f] = c
        with torch.cuda.stream(self.copy):
            for f in coded:
                if lits[f]:
                    dl[f][: lits[f]].copy_(hl[f][: lits[f]], non_blocking=True)
            if coded:
                dc.copy_(hc, non_blocking=True)
                rc = self._decode(coded, dc, offs, dl, vals, dnv)
                _lib.check(rc, "recd_rowcode_decode")
            ev = torch.cuda.Event()
            ev.record(self.copy)
            self._h_done[slot] = ev
            self._pc_done[slot] = ev
            self.ready[slot].record(self.copy)
        self.counts[slot] = n
        self.h2d_bytes[slot] = sum(8 * offs[f].numel() + 8 for f in range(F)) + \
            sum(8 * n[f] for f in raw) + sum(8 * lits[f] + self.step.B for f in coded)

    def _raw_keys(self, n: list) -> set:
        """Keys copied raw: largest first, skipping any that would take the
        raw IDs past raw_share of the batch (so the share is met from below
        to within the smallest key, not overshot by a whole long key)."""
        target = self.raw_share * sum(n)
        raw, acc = set(), 0
        for f in sorted(range(len(n)), key=lambda f: -n[f]):
            if n[f] and acc + n[f] <= target:
                raw.add(f)
                acc += n[f]
        return raw

    def _decode(self, coded, dc, offs, dl, vals, dnv):
        """recd_rowcode_decode over the coded keys (a subset's value counts
        gathered into a contiguous device array first)."""
        nv = dnv
        if len(coded) < len(vals):
            nv = self._nv_sub = dnv.index_select(
                0, torch.tensor(coded, dtype=torch.int64).to(self.dev, non_blocking=True))
        L = _lib.load()
        return L.recd_rowcode_decode(len(coded), self.step.B, _lib.ptrs([dc[f] for f in coded]),
                                     _lib.ptrs([offs[f] for f in coded]), nv.data_ptr(),
                                     _lib.i64s([self._capv[f] for f in coded]),
                                     _lib.ptrs([dl[f] for f in coded]),
                                     _lib.ptrs([vals[f] for f in coded]),
                                     self._rc_scratch.data_ptr(), self._rc_scratch.numel(),
                                     self.copy.cuda_stream)

    def run(self, slot: int, replay) -> None:
        """Run one step on `slot` (after its copy), then hand the slot back to
        the copy stream.  `replay` launches the step (e.g. step.replay)."""
        cur = torch.cuda.current_stream(self.dev)
        cur.wait_event(self.ready[slot])
        if self.direct:
            self.step.use_slot(slot)
            self.step.slot_nvalues[slot] = list(self.counts[slot])
        else:
            self.install(slot, _record=False)
        replay()
        self.free[slot].record(cur)
        self._freed[slot] = True

    def wait_ready(self, slot: int) -> None:
        """The current stream waits for `slot`'s H2D copy (pipelined steps: the
        side stream of the next graph deduplicates that slot)."""
        torch.cuda.current_stream(self.dev).wait_event(self.ready[slot])
        if self.direct:
            self.step.slot_nvalues[slot] = list(self.counts[slot])

    def release(self, slot: int) -> None:
        """Everything enqueued so far on the current stream is done with
        `slot`: the next prefetch into it may start once the stream gets here."""
        self.free[slot].record(torch.cuda.current_stream(self.dev))
        self._freed[slot] = True

    def install(self, slot: int, _record: bool = True) -> None:
        """Copy `slot` into a slot-less step's inputs (on the current stream,
        after its H2D copy)."""
        cur = torch.cuda.current_stream(self.dev)
        cur.wait_event(self.ready[slot])
        vals, offs = self.slots[slot]
        n = self.counts[slot]
        if n != list(self.step.nvalues):
            if getattr(self.step, "graph", None) is not None:
                raise ValueError("batch value counts differ from the captured graph's")
            self.step.nvalues = list(n)
            self.step.a_nvalues = _lib.i64s(n)
        for f in range(len(vals)):
            self.step.in_values[f][: n[f]].copy_(vals[f][: n[f]], non_blocking=True)
            self.step.in_offsets[f].copy_(offs[f], non_blocking=True)
        if _record:
            self.free[slot].record(cur)
            self._freed[slot] = True
