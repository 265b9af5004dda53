"""Deduplicated sequence encoder (config 4): the reference's `attention_pool`
(trainer_sim.py:347-391) evaluated over the UNIQUE rows of a grouped IKJT and
expanded back to the batch by inverse_lookup (trainer_sim.py:558-561).

    out[u] = mean_i softmax(q k^T / sqrt(d))_i v  @ W_o,  q, k, v = x W_{q,k,v}

where x stacks the embedding rows of every feature of the group for unique
row u (empty row -> 0).  The QKV projection over all unique tokens runs on
the tcgen05 tensor cores in BF16 with FP32 accumulation (recd_attention_pool,
csrc/recd_encoder.cu); per-row scores use mma.sync BF16, softmax statistics,
P column sums, the value mix and W_o are FP32.  BF16 operands make the result
differ from the FP32 reference by ~1e-2 relative -- the tolerance the tests
state; the KJT baseline runs the same kernels over all B rows.
"""

from __future__ import annotations

from typing import Sequence

import numpy as np
import torch

from . import _lib
from .embedding import EmbeddingTable
from .tensors import IKJT, KJT

__all__ = ["DedupAttentionPool", "attention_pool_macs"]


def attention_pool_macs(lengths: np.ndarray, d: int) -> int:
    """MAC count of the reference's per-row loop (trainer_sim.py:380-389)."""
    n = np.asarray(lengths, dtype=np.int64)
    n = n[n > 0]
    return int((3 * n * d * d + 2 * n * n * d + d * d).sum())


def _as_f32(w, dev) -> torch.Tensor:
    return torch.as_tensor(np.asarray(w, dtype=np.float32) if not isinstance(w, torch.Tensor) else w,
                           dtype=torch.float32, device=dev)


class DedupAttentionPool:
    """attention_pool over the unique rows of one dedup group."""

    def __init__(self, tables: dict[str, EmbeddingTable], w_q, w_k, w_v, w_o):
        self.tables = dict(tables)
        t0 = next(iter(self.tables.values()))
        self.dev = t0.weights.device
        self.d = t0.dim
        if any(t.dim != self.d for t in self.tables.values()):
            raise ValueError("all tables of a group must share one embedding dim")
        if self.d not in (64, 128):
            raise ValueError(f"encoder supports d in (64, 128), got {self.d}")
        wq, wk, wv = (_as_f32(w, self.dev) for w in (w_q, w_k, w_v))
        # GEMM operand B = [W_q | W_k | W_v]^T, K-major (rows = output features)
        self.w_qkv_t = torch.cat([wq.t(), wk.t(), wv.t()], 0).contiguous().to(torch.bfloat16)
        self.w_o = _as_f32(w_o, self.dev).contiguous()
        self.lib = _lib.load()

    def unique_rows(self, features: Sequence, keys: Sequence[str]) -> torch.Tensor:
        """[U, d] outputs for jagged features sharing U rows (one per key)."""
        F = len(features)
        U = features[0].row_count
        if any(f.row_count != U for f in features):
            raise ValueError("features of a group must have the same row count")
        tabs = [self.tables[k] for k in keys]
        caps = [max(int(f.values.numel()), 1) for f in features]
        counts = torch.tensor([U] * F + [int(f.values.numel()) for f in features],
                              dtype=torch.int64, device=self.dev)
        out = torch.empty((max(U, 1), self.d), dtype=torch.float32, device=self.dev)
        if U == 0:
            return out[:0]
        scratch = _lib.Workspace.get(
            self.lib.recd_attention_pool_scratch_bytes(F, self.d, _lib.i64s(caps)), self.dev, "encoder")
        err = torch.empty(2, dtype=torch.int64, device=self.dev)
        rc = self.lib.recd_attention_pool(
            F, U, self.d, _lib.ptrs([t.weights for t in tabs]), _lib.i64s([t.rows for t in tabs]),
            _lib.ptrs([f.values for f in features]), _lib.ptrs([f.offsets for f in features]),
            _lib.i64s(caps), counts.data_ptr(), self.w_qkv_t.data_ptr(), self.w_o.data_ptr(),
            out.data_ptr(), err.data_ptr(), scratch.data_ptr(), scratch.numel(), _lib.stream_ptr(self.dev))
        _lib.check(rc, "recd_attention_pool")
        e = int(err[0].item())
        if e != _lib.RECD_NO_ERROR:
            f, p = e >> 40, e & ((1 << 40) - 1)
            raise ValueError(f"feature {keys[f]!r}: ID {int(features[f].values[p])} at position {p} "
                             f"out of range [0, {tabs[f].rows})")
        return out

    def __call__(self, x: IKJT | KJT, keys: Sequence[str] | None = None) -> torch.Tensor:
        """IKJT: unique rows, then expansion by inverse_lookup ([B, d]).
        KJT (the baseline path): every batch row is encoded."""
        if isinstance(x, IKJT):
            keys = list(keys or x.group_keys)
            pooled = self.unique_rows([x.per_feature[k] for k in keys], keys)
            out = torch.empty((x.batch_size, self.d), dtype=torch.float32, device=self.dev)
            rc = self.lib.recd_expand(1, x.batch_size, self.d, _lib.ptrs([x.inverse_lookup]),
                                      _lib.ptrs([pooled]), _lib.ptrs([out]), _lib.stream_ptr(self.dev))
            _lib.check(rc, "recd_expand")
            return out
        keys = list(keys or x.keys)
        return self.unique_rows([x.entries[k] for k in keys], keys)
