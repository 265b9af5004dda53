"""Oracle restatement of the reference's jagged / IKJT tensor algorithms.

TEST INFRASTRUCTURE ONLY (see `oracle/__init__.py`).  Every function works
on the reference's array layout: a jagged feature is ``(values int64[N],
offsets int64[R])`` with one offset per row and the last row running to the
end of ``values`` (`tensors.py:60-111`).
"""

from __future__ import annotations

import hashlib
import struct
from typing import Mapping, Sequence

import numpy as np

_I64 = np.dtype("<i8")


def row_lengths(values: np.ndarray, offsets: np.ndarray) -> np.ndarray:
    """`JaggedTensor.row_lengths` (tensors.py:98-100)."""
    bounds = np.append(np.asarray(offsets, dtype=np.int64), np.int64(len(values)))
    return np.diff(bounds)


def _rows(values: np.ndarray, offsets: np.ndarray) -> list[np.ndarray]:
    """`JaggedTensor.row` for every row (tensors.py:102-108)."""
    n = len(offsets)
    out = []
    for i in range(n):
        end = offsets[i + 1] if i + 1 < n else len(values)
        out.append(values[offsets[i]:end])
    return out


def _from_rows(rows: Sequence[np.ndarray]) -> tuple[np.ndarray, np.ndarray]:
    """`JaggedTensor.from_rows` (tensors.py:84-92)."""
    arrs = [np.asarray(r, dtype=np.int64) for r in rows]
    lengths = np.array([a.size for a in arrs], dtype=np.int64)
    offsets = np.zeros(len(arrs), dtype=np.int64)
    if len(arrs) > 1:
        np.cumsum(lengths[:-1], out=offsets[1:])
    values = np.concatenate(arrs) if arrs else np.empty(0, dtype=np.int64)
    return values.astype(np.int64), offsets


def _feature_list(row, key: str) -> np.ndarray:
    """`_row_features` + `_feature_list` (tensors.py:228-243): absent keys are
    empty lists; rows are Mappings or objects with ``.features``."""
    feats = getattr(row, "features", None)
    if feats is None:
        if not isinstance(row, Mapping):
            raise TypeError(f"cannot extract features from {type(row).__name__}")
        feats = row
    seq = feats.get(key)
    if seq is None:
        return np.empty(0, dtype=np.int64)
    return np.asarray(seq, dtype=np.int64)


def build_kjt_arrays(rows: Sequence, keys: Sequence[str]) -> dict[str, tuple[np.ndarray, np.ndarray]]:
    """`build_kjt` (tensors.py:246-254) -> {key: (values, offsets)}."""
    if len(rows) == 0:
        raise ValueError("empty batch")
    return {key: _from_rows([_feature_list(r, key) for r in rows]) for key in keys}


def _pack_group_row(arrs: Sequence[np.ndarray]) -> bytes:
    """`_pack_group_row` (tensors.py:257-262): per feature ``<u32 len>`` then
    the int64 little-endian values."""
    parts = []
    for arr in arrs:
        parts.append(struct.pack("<I", arr.size))
        parts.append(arr.astype(_I64, copy=False).tobytes())
    return b"".join(parts)


def _content_hash(packed: bytes) -> int:
    """`_content_hash` (tensors.py:265-266): blake2b, 8-byte digest."""
    return int.from_bytes(hashlib.blake2b(packed, digest_size=8).digest(), "little")


def _dedup_row_lists(row_lists: list[list[np.ndarray]]):
    """The bucket loop of `build_ikjt` (tensors.py:283-298): content hash ->
    bucket -> full byte compare; uid = first occurrence order."""
    inverse = np.empty(len(row_lists), dtype=np.int64)
    buckets: dict[int, list[tuple[int, bytes]]] = {}
    first_rows: list[int] = []
    for i, arrs in enumerate(row_lists):
        packed = _pack_group_row(arrs)
        bucket = buckets.setdefault(_content_hash(packed), [])
        uid = -1
        for cand_uid, cand_packed in bucket:
            if cand_packed == packed:
                uid = cand_uid
                break
        if uid < 0:
            uid = len(first_rows)
            first_rows.append(i)
            bucket.append((uid, packed))
        inverse[i] = uid
    return inverse, first_rows


def build_ikjt_arrays(features: Sequence[tuple[np.ndarray, np.ndarray]]):
    """`build_ikjt` (tensors.py:269-308) over KJT-form inputs.

    ``features`` is the group's list of (values, offsets), all with B rows.
    Returns ``(inverse int64[B], [(uvalues, uoffsets) per feature])``.
    """
    if len(features) == 0:
        raise ValueError("empty dedup group")
    b = len(features[0][1])
    if b == 0:
        raise ValueError("empty batch")
    per_feat_rows = [_rows(np.asarray(v, dtype=np.int64), np.asarray(o, dtype=np.int64))
                     for v, o in features]
    row_lists = [[rows[i] for rows in per_feat_rows] for i in range(b)]
    inverse, first_rows = _dedup_row_lists(row_lists)
    out = [_from_rows([row_lists[i][k] for i in first_rows]) for k in range(len(features))]
    return inverse, out


def build_ikjt_rows(rows: Sequence, group: Sequence[str]):
    """`build_ikjt(rows, group)` (tensors.py:269-308) over record rows.
    Returns ``(inverse, {key: (uvalues, uoffsets)})``."""
    if len(rows) == 0:
        raise ValueError("empty batch")
    if len(group) == 0:
        raise ValueError("empty dedup group")
    row_lists = [[_feature_list(r, key) for key in group] for r in rows]
    inverse, first_rows = _dedup_row_lists(row_lists)
    per_feature = {
        key: _from_rows([row_lists[i][k] for i in first_rows])
        for k, key in enumerate(group)
    }
    return inverse, per_feature


def jagged_index_select(values: np.ndarray, offsets: np.ndarray, indices) -> tuple[np.ndarray, np.ndarray]:
    """`jagged_index_select` (tensors.py:363-390), same IndexError text."""
    values = np.asarray(values, dtype=np.int64)
    offsets = np.asarray(offsets, dtype=np.int64)
    idx = np.asarray(indices, dtype=np.int64)
    n = len(offsets)
    if idx.size:
        bad = np.flatnonzero((idx < 0) | (idx >= n))
        if bad.size:
            p = int(bad[0])
            raise IndexError(f"index {int(idx[p])} at position {p} out of range for {n} rows")
    lengths = row_lengths(values, offsets)
    sel_len = lengths[idx]
    out_offsets = np.zeros(idx.size, dtype=np.int64)
    if idx.size > 1:
        np.cumsum(sel_len[:-1], out=out_offsets[1:])
    total = int(sel_len.sum())
    gather = np.repeat(offsets[idx] - out_offsets, sel_len) + np.arange(total, dtype=np.int64)
    return values[gather], out_offsets


def ikjt_to_kjt_arrays(inverse: np.ndarray, per_feature: Sequence[tuple[np.ndarray, np.ndarray]]):
    """`ikjt_to_kjt` (tensors.py:393-399): expand every feature by the inverse."""
    return [jagged_index_select(v, o, inverse) for v, o in per_feature]


def slice_ikjt_rows(inverse: np.ndarray, per_feature: Sequence[tuple[np.ndarray, np.ndarray]],
                    start: int, stop: int):
    """`slice_ikjt_rows` (trainer_sim.py:394-413): restrict to rows
    [start, stop) without re-hashing; renumber surviving unique rows in
    first-occurrence order."""
    u = len(per_feature[0][1])
    b = len(inverse)
    if not 0 <= start < stop <= b:
        raise ValueError(f"bad row range [{start}, {stop})")
    inv = np.asarray(inverse, dtype=np.int64)[start:stop]
    uniq, first_idx = np.unique(inv, return_index=True)
    order = uniq[np.argsort(first_idx, kind="stable")]
    lut = np.full(u, -1, dtype=np.int64)
    lut[order] = np.arange(order.size, dtype=np.int64)
    return lut[inv], [jagged_index_select(v, o, order) for v, o in per_feature]
