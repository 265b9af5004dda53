"""Deduplicated pooled embedding lookup (forward + backward) on B200.

Drop-in for the sparse path of `sessiondedup.trainer_sim`
(/root/reference/pkg/src/sessiondedup/trainer_sim.py):

  EmbeddingTable            trainer_sim.py:69-87 (same seeded init via .create)
  embedding_lookup          trainer_sim.py:308-321 -> recd_embedding_lookup
  pool                      trainer_sim.py:324-344 -> recd_pool_dense
  pooled_lookup             lookup + pool + b[inv] (trainer_sim.py:539-561) fused
                            in recd_pool_fwd (activations never materialised)
  pooled_lookup_backward    the backward the reference lacks:
                            recd_pool_bwd, fused SGD or sparse gradients
  DedupEmbeddingBagCollection  nn.Module + autograd over the above
"""

from __future__ import annotations

import hashlib
from typing import Mapping, Sequence

import numpy as np
import torch

from . import _lib
from .tensors import IKJT, KJT, JaggedTensor, default_device

__all__ = [
    "EmbeddingTable",
    "embedding_lookup",
    "pool",
    "pooled_lookup",
    "pooled_lookup_backward",
    "DedupEmbeddingBagCollection",
    "ELEMENT_POOLING",
    "raise_lookup_error",
]

ELEMENT_POOLING = ("sum", "avg", "max")  # trainer_sim.py:58


def _key_seed(base: int, *names: str) -> np.random.Generator:
    """trainer_sim.py:62-66 (same SeedSequence derivation)."""
    tag = hashlib.blake2b("|".join(names).encode("utf-8"), digest_size=8).digest()
    return np.random.default_rng(np.random.SeedSequence((base, int.from_bytes(tag, "little"))))


class EmbeddingTable:
    """fp32 (rows, dim) table on the GPU (trainer_sim.py:69-87)."""

    def __init__(self, key: str, rows: int, dim: int, weights: torch.Tensor):
        if tuple(weights.shape) != (rows, dim):
            raise ValueError("weight shape does not match rows x dim")
        if weights.dtype != torch.float32:
            raise ValueError("weights must be float32")
        _lib.require_cuda(weights)
        self.key, self.rows, self.dim = key, int(rows), int(dim)
        self.weights = weights.contiguous()

    @staticmethod
    def init_weights(key: str, rows: int, dim: int, seed: int) -> np.ndarray:
        """The reference's seeded init (trainer_sim.py:62-66, 83-87): numpy
        uniform(-0.1, 0.1) from SeedSequence((seed, blake2b(key))), host side."""
        rng = _key_seed(seed, "table", key)
        return rng.uniform(-0.1, 0.1, size=(rows, dim)).astype(np.float32)

    @classmethod
    def create(cls, key: str, rows: int, dim: int, seed: int, device=None) -> "EmbeddingTable":
        """Bit-identical to the reference's seeded init (numpy RNG on host)."""
        w = cls.init_weights(key, rows, dim, seed)
        return cls(key, rows, dim, torch.from_numpy(w).to(device or default_device()))

    @classmethod
    def create_on_device(cls, key: str, rows: int, dim: int, seed: int, device=None,
                         chunk_rows: int = 1 << 22) -> "EmbeddingTable":
        """uniform(-0.1, 0.1) drawn on the GPU (for multi-GB tables; not
        bit-identical to the numpy init)."""
        dev = device or default_device()
        w = torch.empty((rows, dim), dtype=torch.float32, device=dev)
        g = torch.Generator(device=dev)
        g.manual_seed(int.from_bytes(hashlib.blake2b(f"{seed}|{key}".encode(), digest_size=8)
                                     .digest(), "little") & ((1 << 63) - 1))
        for r0 in range(0, rows, chunk_rows):
            w[r0:r0 + chunk_rows].uniform_(-0.1, 0.1, generator=g)
        return cls(key, rows, dim, w)


def embedding_lookup(jt: JaggedTensor, table: EmbeddingTable, key: str = "") -> torch.Tensor:
    """One embedding row per value, in values order (trainer_sim.py:308-321)."""
    lib = _lib.load()
    dev = jt.device
    n = jt.values.numel()
    out = torch.empty((n, table.dim), dtype=torch.float32, device=dev)
    err = torch.empty(1, dtype=torch.int64, device=dev)
    rc = lib.recd_embedding_lookup(table.weights.data_ptr(), table.rows, table.dim,
                                   jt.values.data_ptr(), n, out.data_ptr(), err.data_ptr(),
                                   _lib.stream_ptr(dev))
    _lib.check(rc, "recd_embedding_lookup")
    e = int(err.item())
    if e != _lib.RECD_NO_ERROR:
        raise ValueError(f"feature {key or table.key!r}: ID {int(jt.values[e])} at position {e} "
                         f"out of range [0, {table.rows})")
    return out


def pool(activations: torch.Tensor, offsets: torch.Tensor, op: str) -> torch.Tensor:
    """Per-row reduction of materialised activations, empty rows -> 0, sum in
    numpy's reduceat order (trainer_sim.py:324-344)."""
    if op not in ELEMENT_POOLING:
        raise ValueError(f"unknown pooling op {op!r}")
    lib = _lib.load()
    acts = activations.contiguous()
    _lib.require_cuda(acts)
    offs = torch.as_tensor(offsets, dtype=torch.int64, device=acts.device).contiguous()
    out = torch.empty((offs.numel(), acts.shape[1]), dtype=torch.float32, device=acts.device)
    rc = lib.recd_pool_dense(acts.data_ptr(), acts.shape[0], acts.shape[1], offs.data_ptr(),
                             offs.numel(), _lib.POOL_MODES[op], out.data_ptr(),
                             _lib.stream_ptr(acts.device))
    _lib.check(rc, "recd_pool_dense")
    return out


def _counts_tensor(features: Sequence[JaggedTensor], dev) -> torch.Tensor:
    c = [f.row_count for f in features] + [f.values.numel() for f in features]
    return torch.tensor(c, dtype=torch.int64, device=dev)


def pooled_lookup(features: Sequence[JaggedTensor], tables: Sequence[EmbeddingTable], op: str,
                  inverses: Sequence[torch.Tensor | None] | None = None,
                  batch_size: int | None = None, keys: Sequence[str] | None = None,
                  counts: torch.Tensor | None = None, err: torch.Tensor | None = None
                  ) -> list[torch.Tensor]:
    """For each feature f: pool(embedding_lookup(features[f], tables[f]))
    expanded by inverses[f] (None = the rows are the batch rows).  Returns
    one [B, D] tensor per feature.  One fused launch pair for all features.

    The out-of-range check reads one device word back (a host sync).  Pass
    an `err` tensor (int64[2], device) to defer it: nothing is read, the call
    is capturable in a CUDA graph, and `raise_lookup_error(err, ...)` raises
    the reference's ValueError later."""
    if op not in ELEMENT_POOLING:
        raise ValueError(f"unknown pooling op {op!r}")
    lib = _lib.load()
    F = len(features)
    dev = features[0].device
    dims = {t.dim for t in tables}
    if len(dims) != 1:
        raise ValueError("all tables must share one embedding dim")
    D = dims.pop()
    inverses = list(inverses) if inverses is not None else [None] * F
    B = batch_size if batch_size is not None else (
        inverses[0].numel() if inverses[0] is not None else features[0].row_count)
    counts = counts if counts is not None else _counts_tensor(features, dev)
    pooled, outs = [], []
    for f in range(F):
        if inverses[f] is None:
            o = torch.empty((B, D), dtype=torch.float32, device=dev)
            pooled.append(o)
            outs.append(o)
        else:
            pooled.append(torch.empty((max(features[f].row_count, 1), D), dtype=torch.float32,
                                      device=dev))
            outs.append(torch.empty((B, D), dtype=torch.float32, device=dev))
    deferred = err is not None
    if not deferred:
        err = torch.empty(2, dtype=torch.int64, device=dev)  # [first bad ID, work counter]
    rc = lib.recd_pool_fwd(F, B, D, _lib.POOL_MODES[op], _lib.ptrs([t.weights for t in tables]),
                           _lib.i64s([t.rows for t in tables]),
                           _lib.ptrs([f.values for f in features]),
                           _lib.ptrs([f.offsets for f in features]), counts.data_ptr(),
                           _lib.ptrs(inverses), _lib.ptrs(pooled), _lib.ptrs(outs),
                           err.data_ptr(), _lib.stream_ptr(dev))
    _lib.check(rc, "recd_pool_fwd")
    if not deferred:
        raise_lookup_error(err, features, tables, keys)
    return outs


def raise_lookup_error(err: torch.Tensor, features: Sequence[JaggedTensor],
                       tables: Sequence[EmbeddingTable], keys: Sequence[str] | None = None) -> None:
    """Raise the reference's ValueError (trainer_sim.py:312-320) if the lookup
    that wrote `err` saw an ID outside [0, rows) (one host read)."""
    e = int(err[0].item())
    if e != _lib.RECD_NO_ERROR:
        f, p = e >> 40, e & ((1 << 40) - 1)
        key = keys[f] if keys else tables[f].key
        raise ValueError(f"feature {key!r}: ID {int(features[f].values[p])} at position {p} "
                         f"out of range [0, {tables[f].rows})")


def pooled_lookup_backward(features: Sequence[JaggedTensor], tables: Sequence[EmbeddingTable],
                           op: str, grad_outputs: Sequence[torch.Tensor],
                           inverses: Sequence[torch.Tensor | None] | None = None,
                           lr: float | None = None, counts: torch.Tensor | None = None):
    """Backward of `pooled_lookup` (our definition, oracle/embedding.py):
    grad_u = ordered segment-sum of grad_out onto unique rows, then a
    deterministic ID-sorted scatter-add.  With ``lr`` the SGD update
    W[id] -= lr * g is applied in place and None is returned; otherwise a
    list with one ``(ids, grads)`` pair per distinct table (in first-use
    order) is returned."""
    if op not in ("sum", "avg"):
        raise ValueError(f"backward supports sum/avg pooling, got {op!r}")
    lib = _lib.load()
    F = len(features)
    dev = features[0].device
    D = tables[0].dim
    inverses = list(inverses) if inverses is not None else [None] * F
    B = grad_outputs[0].shape[0]
    counts = counts if counts is not None else _counts_tensor(features, dev)
    grads = [g.contiguous() for g in grad_outputs]
    caps = [max(f.values.numel(), 1) for f in features]
    nbytes = lib.recd_pool_bwd_scratch_bytes(F, B, D, _lib.i64s(caps))
    scratch = _lib.Workspace.get(nbytes, dev, "bwd")
    apply = lr is not None
    ids_out, rows_out = [], []
    gcounts = torch.zeros(F, dtype=torch.int64, device=dev)
    if not apply:
        ids_out = [torch.empty(c, dtype=torch.int64, device=dev) for c in caps]
        rows_out = [torch.empty((c, D), dtype=torch.float32, device=dev) for c in caps]
    rc = lib.recd_pool_bwd(F, B, D, _lib.POOL_MODES[op], _lib.ptrs([t.weights for t in tables]),
                           _lib.i64s([t.rows for t in tables]),
                           _lib.ptrs([f.values for f in features]),
                           _lib.ptrs([f.offsets for f in features]), _lib.i64s(caps),
                           counts.data_ptr(), _lib.ptrs(inverses), _lib.ptrs(grads),
                           float(lr or 0.0), 1 if apply else 0,
                           _lib.ptrs(ids_out) if not apply else None,
                           _lib.ptrs(rows_out) if not apply else None,
                           gcounts.data_ptr() if not apply else None,
                           scratch.data_ptr(), scratch.numel(), _lib.stream_ptr(dev))
    _lib.check(rc, "recd_pool_bwd")
    if apply:
        return None
    n = gcounts.cpu().tolist()
    seen, out = set(), []
    for f in range(F):
        ptr = tables[f].weights.data_ptr()
        if ptr in seen:
            continue
        seen.add(ptr)
        out.append((ids_out[f][: n[f]], rows_out[f][: n[f]]))
    return out


class _PooledFn(torch.autograd.Function):
    """Autograd node of one pooled_lookup call; the tables, batch size and
    counts the backward needs are kept on ctx (not on the module), so several
    forwards may be in flight before their backwards run."""

    @staticmethod
    def forward(ctx, anchor, lr, tables, features, inverses, counts, op, B, sink, err):
        outs = pooled_lookup(features, tables, op, inverses, B, counts=counts, err=err)
        ctx.lr, ctx.tables, ctx.features, ctx.inverses, ctx.counts, ctx.op, ctx.B, ctx.sink = (
            lr, tables, features, inverses, counts, op, B, sink)
        return tuple(outs)

    @staticmethod
    def backward(ctx, *grads):
        feats = ctx.features
        dev = feats[0].device
        D = ctx.tables[0].dim
        grads = [g if g is not None else torch.zeros((ctx.B, D), device=dev) for g in grads]
        res = pooled_lookup_backward(feats, ctx.tables, ctx.op, grads, ctx.inverses, lr=ctx.lr,
                                     counts=ctx.counts)
        if res is not None:
            ctx.sink.extend(res)
        return (None,) * 10


class DedupEmbeddingBagCollection(torch.nn.Module):
    """Pooled embedding bags over IKJT groups (sum / avg / max per key; max is
    forward-only -- its outputs carry no autograd graph, and lr with max is
    rejected at construction).

    ``forward`` takes the step's IKJTs (and/or a KJT for plain keys) and
    returns {key: [B, D]} -- each unique row is looked up and pooled once, then
    expanded through its group's inverse_lookup (trainer_sim.py:531-574).
    ``backward`` runs recd_pool_bwd: with ``lr`` set the tables are updated in
    place by fused SGD (like an FBGEMM TBE fused optimizer); with ``lr=None``
    sparse (ids, grads) pairs are collected in ``self.sparse_grads``.
    """

    def __init__(self, tables: Mapping[str, EmbeddingTable], pooling: Mapping[str, str] | str = "sum",
                 lr: float | None = None, defer_checks: bool = False):
        super().__init__()
        self.tables = dict(tables)
        dims = {t.dim for t in self.tables.values()}
        if len(dims) != 1:
            raise ValueError("all tables must share one embedding dim")
        self.dim = dims.pop()
        if isinstance(pooling, str):
            pooling = {k: pooling for k in self.tables}
        for k, op in pooling.items():
            if op not in ELEMENT_POOLING:
                raise ValueError(f"unknown pooling op {op!r}")
        self.pooling = dict(pooling)
        if lr is not None and "max" in self.pooling.values():
            # the fused SGD runs in the backward, which max pooling does not have
            raise ValueError("max pooling is forward-only: it cannot be trained with lr "
                             "(use sum or avg)")
        self.lr = lr
        self.sparse_grads: list = []
        self._anchor = torch.nn.Parameter(torch.zeros(0))
        # defer_checks: forward never reads the device (capturable); check() raises
        self.defer_checks = bool(defer_checks)
        self._pending: list = []   # (err, features, tables, keys) of deferred lookups

    def forward(self, ikjts: Sequence[IKJT] = (), kjt: KJT | None = None) -> dict[str, torch.Tensor]:
        if isinstance(ikjts, IKJT):
            ikjts = [ikjts]
        jobs = []  # (key, feature, inverse)
        B = None
        for ik in ikjts:
            B = ik.batch_size
            for k in ik.group_keys:
                jobs.append((k, ik.per_feature[k], ik.inverse_lookup))
        if kjt is not None:
            B = kjt.batch_size
            for k, jt in kjt.entries.items():
                jobs.append((k, jt, None))
        if not jobs:
            return {}
        out: dict[str, torch.Tensor] = {}
        by_op: dict[str, list] = {}
        for job in jobs:
            if job[0] not in self.tables:
                raise ValueError(f"feature {job[0]!r} has no table")
            by_op.setdefault(self.pooling.get(job[0], "sum"), []).append(job)
        for op, js in by_op.items():
            feats = [j[1] for j in js]
            tables = [self.tables[j[0]] for j in js]
            counts = _counts_tensor(feats, feats[0].device)
            invs = [j[2] for j in js]
            err = None
            if self.defer_checks:
                err = torch.empty(2, dtype=torch.int64, device=feats[0].device)
                self._pending.append((err, feats, tables, [j[0] for j in js]))
            if op == "max":   # forward-only (no backward exists for max): no autograd node
                res = pooled_lookup(feats, tables, op, invs, B, counts=counts, err=err)
            else:
                res = _PooledFn.apply(self._anchor, self.lr, tables, feats, invs, counts, op, B,
                                      self.sparse_grads, err)
            for j, r in zip(js, res):
                out[j[0]] = r
        return out

    def check(self) -> None:
        """Raise the first deferred lookup error (defer_checks=True), in call
        order, and forget the checked lookups.  The fused SGD of a batch with
        an out-of-range ID updates nothing (the backward skips it)."""
        pending, self._pending = self._pending, []
        for err, feats, tables, keys in pending:
            raise_lookup_error(err, feats, tables, keys)
