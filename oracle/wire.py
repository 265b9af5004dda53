"""Restatement of the canonical wire format -- TEST INFRASTRUCTURE ONLY (see
oracle/__init__.py).

`/root/reference/pkg/src/sessiondedup/tensors.py:463-515`, little-endian:
  u32 key count; per key: u32 byte length + UTF-8 bytes
  u64 batch size B
  u8 inverse flag; if 1, B x i64 inverse_lookup
  per key: u64 offsets count + i64 offsets
  per key: u64 values count + i64 values
slice_stream_bytes = 16 + 8 (|offsets| + |values|); values_stream_bytes = 8 |values|.
Pinned by tests/golden/wire.npz (bytes of the real serialize_kjt / serialize_ikjt).
"""

from __future__ import annotations

import struct
from typing import Sequence

import numpy as np


def serialize(keys: Sequence[str], batch_size: int, inverse, offsets: Sequence[np.ndarray],
              values: Sequence[np.ndarray]) -> bytes:
    parts = [struct.pack("<I", len(keys))]
    for k in keys:
        kb = k.encode("utf-8")
        parts += [struct.pack("<I", len(kb)), kb]
    parts.append(struct.pack("<Q", batch_size))
    if inverse is None:
        parts.append(b"\x00")
    else:
        parts += [b"\x01", np.asarray(inverse, dtype="<i8").tobytes()]
    for o in offsets:
        parts += [struct.pack("<Q", len(o)), np.asarray(o, dtype="<i8").tobytes()]
    for v in values:
        parts += [struct.pack("<Q", len(v)), np.asarray(v, dtype="<i8").tobytes()]
    return b"".join(parts)


def slice_stream_bytes(offsets, values) -> int:
    return 16 + 8 * (len(offsets) + len(values))


def values_stream_bytes(values) -> int:
    return 8 * len(values)
