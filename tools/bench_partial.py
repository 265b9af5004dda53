"""Partial (shift-aware) IKJT measurement: recd_partial_ikjt over one
session-clustered key at B = 65,536 (cfg2's row lengths 32 and 256), vs the
reference's greedy encoder restated in oracle/partial.py timed on the host
over a bounded sample of rows.  Prints one JSON line.

    python tools/bench_partial.py [--steps 10] [--batch 65536]
"""

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2211_05239_b200 as R  # noqa: E402
from tools.datagen import (FeatureSpec, SampleCountDist, SessionConfig,  # noqa: E402
                                           generate_clustered_batch)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=65536)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--cpu-rows", type=int, default=4096)
    args = ap.parse_args()
    B = args.batch
    torch.cuda.set_device(0)
    out = {"metric": "rows/sec for the partial IKJT (build_partial_ikjt) of one key", "batch": B, "keys": {}}
    for L in (32, 256):
        spec = FeatureSpec("hist", "user_sequence", float(L), 10_000_000, 0.15)
        batch = generate_clustered_batch(SessionConfig(B // 8, SampleCountDist("geometric", 16.5), 0), [spec], B)
        kjt = R.KJT(B, {"hist": R.JaggedTensor(batch.values["hist"], batch.offsets["hist"])})
        ik = R.kjt_to_ikjt(kjt, ["hist"])
        for _ in range(3):
            pk = R.kjt_to_partial_ikjt(kjt, "hist", ik)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            pk = R.kjt_to_partial_ikjt(kjt, "hist", ik)
        torch.cuda.synchronize()
        ms_partial = (time.perf_counter() - t0) * 1e3 / args.steps
        for i in range(args.steps + 3):
            if i == 3:
                torch.cuda.synchronize()
                t0 = time.perf_counter()
            ik2 = R.kjt_to_ikjt(kjt, ["hist"])
            pk = R.kjt_to_partial_ikjt(kjt, "hist", ik2)
        torch.cuda.synchronize()
        ms_total = (time.perf_counter() - t0) * 1e3 / args.steps
        n_ids = int(kjt.entries["hist"].values.numel())
        n_u = int(ik.per_feature["hist"].values.numel())
        # reference arm: the greedy encoder (oracle restatement) on the first rows
        from oracle.partial import build_partial_jagged
        nr = min(args.cpu_rows, B)
        v = batch.values["hist"]
        o = batch.offsets["hist"]
        end = int(o[nr]) if nr < B else v.size
        t0 = time.perf_counter()
        build_partial_jagged(v[:end], o[:nr])
        cpu_s = time.perf_counter() - t0
        out["keys"][f"len{L}"] = {
            "ms_partial_from_ikjt": ms_partial, "ms_dedup_plus_partial": ms_total,
            "rows_per_s": B / (ms_total * 1e-3), "rounds": pk.rounds,
            "ids": n_ids, "exact_dedup_values": n_u, "partial_values": int(pk.values.numel()),
            "cpu_oracle": {"rows": nr, "s": cpu_s, "rows_per_s": nr / cpu_s, "cores": 1,
                           "kind": "port", "note": "grows superlinearly with rows (buffer search)"}}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
