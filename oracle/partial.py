"""Restatement of the partial (shift-aware) IKJT encoder -- TEST
INFRASTRUCTURE ONLY (see oracle/__init__.py).

`build_partial_ikjt` (/root/reference/pkg/src/sessiondedup/tensors.py:311-338,
helpers 341-360), one feature, batch order, one shared int64 value buffer:
  * an empty list gets the window (0, 0) and touches nothing (324-326);
  * else, if the list occurs in the buffer at an element-aligned position,
    the LEFTMOST such position is reused, nothing appended (327-330, 341-349);
  * else the longest k <= min(n - 1, |buffer|) with buffer[-k:] == list[:k]
    is found (longest first, 352-360), list[k:] is appended and the window is
    (|buffer| - k, n) (331-334).
Windows are (offset, length) pairs per batch row; values is the buffer.
Pinned by tests/golden/partial.npz (outputs of the real build_partial_ikjt).
"""

from __future__ import annotations

from typing import Sequence

import numpy as np


def _leftmost(buf: np.ndarray, blen: int, row: np.ndarray) -> int:
    """Leftmost p with buf[p:p+n] == row inside buf[:blen], or -1."""
    n = row.size
    if n > blen:
        return -1
    cand = np.flatnonzero(buf[: blen - n + 1] == row[0])
    for p in cand:
        if np.array_equal(buf[p:p + n], row):
            return int(p)
    return -1


def _suffix_overlap(buf: np.ndarray, blen: int, row: np.ndarray) -> int:
    for k in range(min(row.size - 1, blen), 0, -1):
        if buf[blen - k] == row[0] and np.array_equal(buf[blen - k:blen], row[:k]):
            return k
    return 0


def build_partial(lists: Sequence[np.ndarray]) -> tuple[np.ndarray, np.ndarray]:
    """lists: one int64 array per batch row -> (values, windows[B, 2])."""
    if len(lists) == 0:
        raise ValueError("empty batch")
    cap = int(sum(np.asarray(x).size for x in lists))
    buf = np.empty(max(cap, 1), dtype=np.int64)
    blen = 0
    windows = np.zeros((len(lists), 2), dtype=np.int64)
    for i, x in enumerate(lists):
        row = np.asarray(x, dtype=np.int64)
        n = row.size
        if n == 0:
            continue
        p = _leftmost(buf, blen, row)
        if p >= 0:
            windows[i] = (p, n)
            continue
        k = _suffix_overlap(buf, blen, row)
        buf[blen:blen + n - k] = row[k:]
        windows[i] = (blen - k, n)
        blen += n - k
    return buf[:blen].copy(), windows


def build_partial_jagged(values: np.ndarray, offsets: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """Same, on one key's jagged (values, row-start offsets) (tensors.py:228-254 layout)."""
    values = np.asarray(values, dtype=np.int64)
    offsets = np.asarray(offsets, dtype=np.int64)
    ends = np.append(offsets[1:], values.size)
    return build_partial([values[s:e] for s, e in zip(offsets, ends)])
