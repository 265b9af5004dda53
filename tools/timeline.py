"""Stream timeline of one eager, overlapped cfg2 TrainStep (GPU box):
CUDA events between the library calls on the main and side streams, all
relative to the step start, averaged over a few steps.

    python tools/timeline.py [--config cfg2] [--steps 5]
"""

from __future__ import annotations

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402


def main() -> None:
    import torch

    import paper_2211_05239_b200 as R
    from paper_2211_05239_b200 import _lib as L
    from paper_2211_05239_b200.step import TrainStep

    args = bench.parse(sys.argv[1:])
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    batch = bench.make_batch(args, 0, 1)
    keys = list(batch.keys)
    tables = {k: R.EmbeddingTable.create_on_device(k, args.rows, args.dim, seed=i, device=dev)
              for i, k in enumerate(keys)}
    caps = {k: batch.values[k].size for k in keys}
    step = TrainStep([[k] for k in keys], args.batch, caps, tables, "sum", args.lr, "dedup", dev,
                     overlap=True, slots=1)
    step.load_batch(batch.values, batch.offsets, slot=0)
    step.fill_grad_out(1)
    main_s = torch.cuda.current_stream(dev)
    side = step._side
    names = ["dedup", "pool", "expand", "grad", "scatter", "side_start", "inverse", "occurrences"]
    acc = {n: [] for n in names}
    for it in range(3 + args.steps):
        ev = {n: torch.cuda.Event(enable_timing=True) for n in ["t0"] + names}
        ms, ss = main_s.cuda_stream, side.cuda_stream
        ev["t0"].record(main_s)
        step.dedup(ms)
        ev["dedup"].record(main_s)
        step._ev_fork.record(main_s)
        side.wait_event(step._ev_fork)
        ev["side_start"].record(side)
        step.backward_stages(L.BWD_INVERSE, ss)
        ev["inverse"].record(side)
        step.backward_stages(L.BWD_OCCURRENCES, ss)
        ev["occurrences"].record(side)
        step.forward(ms, share=True)
        ev["pool"].record(main_s)
        step.expand(ms)
        ev["expand"].record(main_s)
        main_s.wait_event(ev["inverse"])
        step.backward_stages(L.BWD_GRAD, ms)
        ev["grad"].record(main_s)
        main_s.wait_event(ev["occurrences"])
        step.backward_stages(L.BWD_SCATTER, ms)
        ev["scatter"].record(main_s)
        torch.cuda.synchronize()
        if it >= 3:
            for n in names:
                acc[n].append(ev["t0"].elapsed_time(ev[n]))
    for n in names:
        v = sorted(acc[n])[len(acc[n]) // 2]
        print(f"{n:12s} ends at {v:7.3f} ms")


if __name__ == "__main__":
    main()
