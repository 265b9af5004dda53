"""Config 4 measurement: dedup'd sequence encoder (attention_pool over the
unique rows of a 2-key synced history group, then inverse expansion) vs the
KJT baseline (every batch row encoded), B=65536, len 32 per key, D=128,
synthetic sessions (mean 16.5, change 0.15).  Prints one JSON line with
samples/s of both paths, the dedup speedup and the tcgen05 QKV GEMM's
tensor-core throughput (TFLOP/s vs MEASURED_PEAKS bf16).

    python tools/bench_encoder.py [--steps 20] [--batch 65536]
"""

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2211_05239_b200 as R  # noqa: E402
from paper_2211_05239_b200 import _lib  # noqa: E402
from tools.datagen import (FeatureSpec, SampleCountDist, SessionConfig,  # noqa: E402
                                           generate_clustered_batch)


def timed(fn, steps):
    s = torch.cuda.current_stream()
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(steps):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=65536)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--dim", type=int, default=128)
    ap.add_argument("--len", type=int, default=32)
    ap.add_argument("--vocab", type=int, default=10_000_000)
    args = ap.parse_args()
    B, D = args.batch, args.dim
    torch.cuda.set_device(0)
    keys = ["hist_a", "hist_b"]
    specs = [FeatureSpec(k, "user_sequence", float(args.len), args.vocab, 0.15, sync_group="hist")
             for k in keys]
    batch = generate_clustered_batch(SessionConfig(B // 8, SampleCountDist("geometric", 16.5), 0), specs, B)
    g = torch.Generator(device="cuda").manual_seed(0)
    tables = {k: R.EmbeddingTable(k, args.vocab, D,
                                  torch.empty((args.vocab, D), device="cuda").uniform_(-0.1, 0.1, generator=g))
              for k in keys}
    rng = np.random.default_rng(0)
    ws = [rng.standard_normal((D, D)).astype(np.float32) / np.sqrt(D) for _ in range(4)]
    enc = R.DedupAttentionPool(tables, *ws)
    kjt = R.KJT(B, {k: R.JaggedTensor(batch.values[k], batch.offsets[k]) for k in keys})
    ik = R.kjt_to_ikjt(kjt, keys)
    U = ik.unique_count
    ntok_u = sum(int(ik.per_feature[k].values.numel()) for k in keys)
    ntok_b = sum(int(kjt.entries[k].values.numel()) for k in keys)

    ms_dedup = timed(lambda: enc(R.kjt_to_ikjt(kjt, keys)), args.steps)
    ms_enc_u = timed(lambda: enc(ik), args.steps)
    ms_kjt = timed(lambda: enc(kjt), args.steps)
    out_u, out_b = enc(ik), enc(kjt)
    bit_exact = bool(torch.equal(out_u, out_b))

    # the QKV projection alone on the unique tokens: tcgen05 GEMM throughput
    lib = _lib.load()
    a = torch.randn(ntok_u, D, device="cuda").to(torch.bfloat16)
    c = torch.empty(ntok_u, 3 * D, device="cuda", dtype=torch.bfloat16)
    mc = torch.tensor([ntok_u], dtype=torch.int64, device="cuda")
    ms_gemm = timed(lambda: lib.recd_gemm_bf16_tn(3 * D, D, a.data_ptr(), enc.w_qkv_t.data_ptr(), c.data_ptr(),
                                                  mc.data_ptr(), _lib.stream_ptr()), args.steps)
    flops = 2.0 * ntok_u * D * 3 * D
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    bf16_peak = peaks.get("bf16_tflops_sustained") or peaks.get("bf16_tflops")
    gemm_bytes = ntok_u * D * 2 + ntok_u * 3 * D * 2
    hbm = peaks.get("hbm_gbs")
    print(json.dumps({
        "metric": "samples/sec for dedup'd sequence encoder (attention_pool over unique rows + expand)",
        "config": {"workload": "cfg4: 2 synced history keys, len 32 each, attention_pool over unique rows",
                   "batch": B, "dim": D, "vocab": args.vocab, "samples_per_session": 16.5, "change_prob": 0.15},
        "U": U, "tokens_unique": ntok_u, "tokens_kjt": ntok_b,
        "dedup_e2e_device": {"ms": ms_dedup, "samples_per_s": B / ms_dedup * 1e3,
                             "what": "kjt_to_ikjt + encoder over unique rows + expand"},
        "encoder_unique": {"ms": ms_enc_u, "samples_per_s": B / ms_enc_u * 1e3},
        "kjt_baseline": {"ms": ms_kjt, "samples_per_s": B / ms_kjt * 1e3},
        "speedup_vs_kjt": ms_kjt / ms_dedup,
        "dedup_equals_kjt_bit_exact": bit_exact,
        "qkv_gemm_tcgen05": {"ms": ms_gemm, "tflops": flops / ms_gemm / 1e9, "peak_tflops": bf16_peak,
                             "frac": (flops / ms_gemm / 1e9 / bf16_peak) if bf16_peak else None,
                             "hbm_gbs": gemm_bytes / ms_gemm / 1e6, "hbm_frac": (gemm_bytes / ms_gemm / 1e6 / hbm)
                             if hbm else None,
                             "bound": "hbm (K = 128: 2*K/(2+6) = 32 FLOP/byte)"},
    }))


if __name__ == "__main__":
    main()
