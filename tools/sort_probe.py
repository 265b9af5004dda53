"""Probe (GPU box): one-sweep sort time by input pattern -- uniform random
24-bit keys vs session-history keys (rows of 256 IDs in shifted-window chains,
the occurrence sort's input order) vs the same keys already sorted.  26
segments x ~1.04 M pairs (cfg2's occurrence sort).  python tools/sort_probe.py"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2211_05239_b200 import _lib  # noqa: E402

lib = _lib.load()
rng = np.random.default_rng(0)
nseg, per, L = 26, 1_040_000, 256


def history(n):
    out, cur = [], list(rng.integers(0, 10_000_000, L))
    while sum(len(r) for r in out) < n:
        out.append(cur)
        cur = list(rng.integers(0, 10_000_000, L)) if rng.random() < 0.3 else cur[1:] + [int(rng.integers(0, 10_000_000))]
    return np.array([v for r in out for v in r][:n], np.uint32)


pats = {"uniform": np.concatenate([rng.integers(0, 10_000_000, per).astype(np.uint32) for _ in range(nseg)]),
        "history": np.concatenate([history(per) for _ in range(nseg)])}
pats["sorted"] = np.concatenate([np.sort(pats["history"][s * per:(s + 1) * per], kind="stable") for s in range(nseg)])
dev = torch.device("cuda")
bases = [s * per for s in range(nseg)]
caps = [per] * nseg
cnt = [torch.tensor([per], dtype=torch.int64, device=dev) for _ in range(nseg)]
nb = lib.recd_sort_pairs_scratch_bytes(nseg, _lib.i64s(bases), _lib.i64s(caps))
scratch = torch.empty(nb, dtype=torch.uint8, device=dev)
alt = (__import__("ctypes").c_int32 * 1)()
for name, k in pats.items():
    ts = []
    for it in range(6):
        kd = torch.from_numpy(k.view(np.int32)).to(dev)
        vd = torch.arange(k.size, dtype=torch.int32, device=dev)
        k2, v2 = torch.empty_like(kd), torch.empty_like(vd)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rc = lib.recd_sort_pairs(nseg, _lib.i64s(bases), _lib.i64s(caps), _lib.ptrs(cnt), 24,
                                 kd.data_ptr(), vd.data_ptr(), k2.data_ptr(), v2.data_ptr(), alt,
                                 scratch.data_ptr(), nb, torch.cuda.current_stream().cuda_stream)
        e1.record()
        torch.cuda.synchronize()
        assert rc == 0
        if it:
            ts.append(e0.elapsed_time(e1))
    print(name, "sort ms", round(min(ts), 3), round(float(np.median(ts)), 3))
