"""Restatement of the reader's element-wise ID transforms -- TEST
INFRASTRUCTURE ONLY (see oracle/__init__.py).

`/root/reference/pkg/src/sessiondedup/reader.py`:
  * `_splitmix64_vec` (reader.py:70-75): z = x + 0x9E3779B97F4A7C15 (uint64),
    two xor-shift-multiply rounds, final xor-shift;
  * `apply_transform` (reader.py:78-83): identity; mod_hash = splitmix64(x)
    mod param as int64; clamp = np.clip(x, 0, param).
Pinned by tests/golden/transforms.npz (made by importing the real reader).
"""

from __future__ import annotations

import numpy as np

_U64 = np.uint64


def splitmix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = np.asarray(x).astype(_U64) + _U64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> _U64(30))) * _U64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> _U64(27))) * _U64(0x94D049BB133111EB)
        return z ^ (z >> _U64(31))


def apply_transform(values: np.ndarray, op: str, param: int | None = None) -> np.ndarray:
    if op == "identity":
        return np.asarray(values)
    if op == "mod_hash":
        return (splitmix64(values) % _U64(param)).astype(np.int64)
    if op == "clamp":
        return np.clip(np.asarray(values), 0, param)
    raise ValueError(f"unknown transform op {op!r}")
