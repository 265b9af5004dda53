"""Double-buffered host -> device staging of KJT batches.

The KJT of a cfg2 batch is ~1 GB of int64 per GPU, so end to end the step is
bound by the PCIe copy, not by the kernels.  `H2DPipeline` copies batch i+1
from pinned host memory into one of two device staging slots on a dedicated
copy stream while step i runs, then installs it into the step's input
buffers with one device-to-device copy (the CUDA graph stays bound to those
buffers).  Works with TrainStep, ShardedTrainStep and PeerShardedStep (any
object with `keys`, `in_values`, `in_offsets`, `nvalues`).
"""

from __future__ import annotations

import torch

from . import _lib

__all__ = ["H2DPipeline"]


class H2DPipeline:
    def __init__(self, step, device=None):
        self.step = step
        self.dev = device or step.in_values[0].device
        self.copy = torch.cuda.Stream(self.dev)
        self.slots = [([torch.empty_like(v) for v in step.in_values],
                       [torch.empty_like(o) for o in step.in_offsets]) for _ in range(2)]
        self.counts = [None, None]
        self.ready = [torch.cuda.Event() for _ in range(2)]
        self.free = [torch.cuda.Event() for _ in range(2)]
        self._freed = [False, False]

    def prefetch(self, slot: int, values: dict, offsets: dict) -> None:
        """Queue the H2D copy of one batch (pinned host tensors) into `slot`."""
        vals, offs = self.slots[slot]
        n = []
        with torch.cuda.stream(self.copy):
            if self._freed[slot]:
                self.copy.wait_event(self.free[slot])
            for f, k in enumerate(self.step.keys):
                v = values[k]
                if v.numel() > vals[f].numel():
                    raise ValueError(f"feature {k!r}: batch exceeds the step's capacity")
                vals[f][: v.numel()].copy_(v, non_blocking=True)
                offs[f].copy_(offsets[k], non_blocking=True)
                n.append(v.numel())
            self.ready[slot].record(self.copy)
        self.counts[slot] = n

    def install(self, slot: int) -> None:
        """Make `slot` the step's input (on the current stream, after its copy)."""
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
        self.free[slot].record(cur)
        self._freed[slot] = True
