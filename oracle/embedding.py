"""Oracle restatement of the reference's embedding lookup / pooling path,
plus our definition of its backward (the reference has none).

TEST INFRASTRUCTURE ONLY (see `oracle/__init__.py`).
"""

from __future__ import annotations

import math
from typing import Sequence

import numpy as np

ELEMENT_POOLING = ("sum", "avg", "max")  # trainer_sim.py:58


def embedding_lookup(values: np.ndarray, weights: np.ndarray, key: str = "") -> np.ndarray:
    """`embedding_lookup` (trainer_sim.py:308-321): one row per value, with
    the reference's out-of-range ValueError text."""
    vals = np.asarray(values, dtype=np.int64)
    rows = weights.shape[0]
    if vals.size:
        bad = np.flatnonzero((vals < 0) | (vals >= rows))
        if bad.size:
            p = int(bad[0])
            raise ValueError(
                f"feature {key!r}: ID {int(vals[p])} at position {p} out of range [0, {rows})"
            )
    return weights[vals]


def pool(activations: np.ndarray, offsets: np.ndarray, op: str) -> np.ndarray:
    """`pool` (trainer_sim.py:324-344): per-row reduceat; empty rows -> 0.

    numpy's ``add.reduceat`` sums a row as ``a[0] + pairwise(a[1:])`` (the
    8-accumulator / 128-block pairwise tree); avg divides by fp32(len)."""
    if op not in ELEMENT_POOLING:
        raise ValueError(f"unknown pooling op {op!r}")
    offsets = np.asarray(offsets, dtype=np.int64)
    n_rows = offsets.size
    dim = activations.shape[1]
    bounds = np.append(offsets, activations.shape[0])
    lengths = np.diff(bounds)
    out = np.zeros((n_rows, dim), dtype=np.float32)
    nonempty = lengths > 0
    if nonempty.any():
        starts = bounds[:-1][nonempty]
        ufunc = np.maximum if op == "max" else np.add
        out[nonempty] = ufunc.reduceat(activations, starts, axis=0)
        if op == "avg":
            out[nonempty] /= lengths[nonempty].astype(np.float32)[:, None]
    return out


def pooled_lookup(values, offsets, weights, op: str, key: str = "") -> np.ndarray:
    """lookup + pool over one jagged feature (trainer_sim.py:539-555)."""
    return pool(embedding_lookup(values, weights, key), offsets, op)


def expand(pooled: np.ndarray, inverse: np.ndarray) -> np.ndarray:
    """Inverse-index expansion ``b[inv]`` (trainer_sim.py:558-561)."""
    return pooled[np.asarray(inverse, dtype=np.int64)]


# ---------------------------------------------------------------------------
# Backward: NOT in the reference ("GPU kernels ... OUT OF SCOPE";
# SURVEY.md §8(a) row a18).  Definition used by the CUDA path:
#   grad_u[u]  = sum_{i: inv[i]=u} grad_out[i], sequential fp32 from +0.0 in
#                ascending i (== np.add.at order);
#   avg        : every element of row u receives grad_u[u] / fp32(len_u);
#   max        : the first position attaining the max (per dim) receives grad_u;
#   grad_W[id] = sequential fp32 sum over the occurrences of id in ascending
#                (unique row, position) order (== np.add.at order);
#   SGD        : W[id] <- W[id] - fp32(lr * grad_W[id])  (no FMA contraction).
# ---------------------------------------------------------------------------


def pool_backward(grad_out: np.ndarray, inverse: np.ndarray | None, num_unique: int) -> np.ndarray:
    """grad_u[U, D] = segment-sum of grad_out rows onto unique rows."""
    grad_out = np.asarray(grad_out, dtype=np.float32)
    if inverse is None:
        return grad_out.copy()
    gu = np.zeros((num_unique, grad_out.shape[1]), dtype=np.float32)
    np.add.at(gu, np.asarray(inverse, dtype=np.int64), grad_out)
    return gu


def _element_grads(grad_u: np.ndarray, values: np.ndarray, offsets: np.ndarray, op: str,
                   weights: np.ndarray | None = None) -> np.ndarray:
    """Per-value gradient contribution [N, D] in values order."""
    values = np.asarray(values, dtype=np.int64)
    lengths = np.diff(np.append(np.asarray(offsets, dtype=np.int64), values.size))
    rowid = np.repeat(np.arange(len(lengths)), lengths)
    if op == "sum":
        return grad_u[rowid]
    if op == "avg":
        scaled = grad_u.copy()
        nz = lengths > 0
        scaled[nz] = grad_u[nz] / lengths[nz].astype(np.float32)[:, None]
        return scaled[rowid]
    if op == "max":
        if weights is None:
            raise ValueError("max backward needs the table weights")
        acts = weights[values]
        contrib = np.zeros_like(acts)
        for u, (s, n) in enumerate(zip(np.asarray(offsets), lengths)):
            if n == 0:
                continue
            arg = np.argmax(acts[s:s + n], axis=0)  # first index on ties
            contrib[s + arg, np.arange(acts.shape[1])] = grad_u[u]
        return contrib
    raise ValueError(f"unknown pooling op {op!r}")


def sparse_table_grad(grad_u: np.ndarray, values: np.ndarray, offsets: np.ndarray, op: str,
                      weights: np.ndarray | None = None):
    """Deterministic sorted scatter-add: returns (ids ascending, grad rows)."""
    values = np.asarray(values, dtype=np.int64)
    contrib = _element_grads(grad_u, values, offsets, op, weights)
    ids, inv_ids = np.unique(values, return_inverse=True)
    g = np.zeros((ids.size, grad_u.shape[1]), dtype=np.float32)
    np.add.at(g, inv_ids, contrib)
    return ids, g


def sgd_apply(weights: np.ndarray, ids: np.ndarray, grads: np.ndarray, lr: float) -> np.ndarray:
    """W[id] <- W[id] - fp32(lr * g), separately rounded (returns a copy)."""
    w = np.array(weights, dtype=np.float32, copy=True)
    w[ids] = w[ids] - (np.float32(lr) * grads).astype(np.float32)
    return w


def attention_pool(per_key: Sequence[tuple[np.ndarray, np.ndarray]], w_q, w_k, w_v, w_o):
    """`attention_pool` (trainer_sim.py:347-391): single-head SDPA over each
    row's concatenated group sequence, mean over the sequence, then @ W_o."""
    n_rows = per_key[0][1].size
    d = w_q.shape[0]
    scale = np.float32(1.0 / math.sqrt(d))
    out = np.zeros((n_rows, d), dtype=np.float32)
    macs = 0
    all_bounds = [(a, np.append(o, a.shape[0])) for a, o in per_key]
    for i in range(n_rows):
        segs = [a[b[i]:b[i + 1]] for a, b in all_bounds]
        x = segs[0] if len(segs) == 1 else np.concatenate(segs, axis=0)
        n = x.shape[0]
        if n == 0:
            continue
        q = x @ w_q
        k = x @ w_k
        v = x @ w_v
        scores = (q @ k.T) * scale
        scores -= scores.max(axis=1, keepdims=True)
        np.exp(scores, out=scores)
        scores /= scores.sum(axis=1, keepdims=True)
        ctx = scores @ v
        out[i] = ctx.mean(axis=0) @ w_o
        macs += 3 * n * d * d + 2 * n * n * d + d * d
    return out, macs
