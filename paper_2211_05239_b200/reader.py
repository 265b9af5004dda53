"""Element-wise ID transforms of the reader, applied on the GPU.

Mirrors `sessiondedup.reader` (`/root/reference/pkg/src/sessiondedup/reader.py`):
`Transform` (reader.py:54-67), `apply_transform` (reader.py:78-83) and the
transform stage of `process` (reader.py:178-217): an IKJT feature is
transformed on its deduplicated values only and stays an IKJT, so the work
shrinks by the dedupe factor and commutes with the expansion
(test_reader.py:176-187).  All transforms of one call are one launch
(`recd_transform`).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Mapping, Sequence

import torch

from . import _lib
from .tensors import IKJT, KJT, JaggedTensor

__all__ = ["Transform", "apply_transform", "process"]

_OPS = {"identity": 0, "mod_hash": 1, "clamp": 2}


@dataclass(frozen=True)
class Transform:
    """Element-wise ID map applied to one feature's values (reader.py:54-67)."""

    op: str  # "identity" | "mod_hash" | "clamp"
    key: str
    param: int | None = None

    def __post_init__(self) -> None:
        if self.op not in _OPS:
            raise ValueError(f"unknown transform op {self.op!r}")
        if self.op in ("mod_hash", "clamp") and (self.param is None or self.param < 1):
            raise ValueError(f"{self.op} needs a positive param")


def _run(pairs: Sequence[tuple[torch.Tensor, Transform]]) -> list[torch.Tensor]:
    """One launch: out_i = transform_i(values_i) (new tensors; inputs untouched)."""
    if not pairs:
        return []
    lib = _lib.load()
    ins = [v for v, _ in pairs]
    outs = [torch.empty_like(v) for v in ins]
    rc = lib.recd_transform(len(pairs), _lib.ptrs(ins), _lib.ptrs(outs),
                            _lib.i64s([v.numel() for v in ins]), None,
                            _lib.i32s([_OPS[t.op] for _, t in pairs]),
                            _lib.i64s([t.param or 0 for _, t in pairs]),
                            _lib.stream_ptr(ins[0].device))
    _lib.check(rc, "recd_transform")
    return outs


def apply_transform(values: torch.Tensor | JaggedTensor, t: Transform):
    """reader.apply_transform on device int64 values (or a JaggedTensor)."""
    if isinstance(values, JaggedTensor):
        if t.op == "identity":
            return values
        return JaggedTensor(_run([(values.values, t)])[0], values.offsets, validate=False)
    _lib.require_cuda(values)
    if t.op == "identity":
        return values
    return _run([(values, t)])[0]


def process(kjts: Mapping[str, JaggedTensor], ikjts: Sequence[IKJT],
            transforms: Sequence[Transform]) -> tuple[dict[str, JaggedTensor], list[IKJT]]:
    """The transform stage of reader.process (reader.py:178-217): transforms of
    a key run in order; IKJT features are transformed on their unique values
    and the inverse is kept.  Raises like the reference for unknown keys."""
    known = set(kjts) | {k for ik in ikjts for k in ik.group_keys}
    by_key: dict[str, list[Transform]] = {}
    for t in transforms:
        if t.key not in known:
            raise ValueError(f"transform targets missing key {t.key!r}")
        by_key.setdefault(t.key, []).append(t)
    cur: dict[tuple, JaggedTensor] = {("k", k): jt for k, jt in kjts.items()}
    for i, ik in enumerate(ikjts):
        for k, jt in ik.per_feature.items():
            cur[("i", i, k)] = jt
    depth = max((len(v) for v in by_key.values()), default=0)
    for level in range(depth):  # one launch per transform depth across all features
        slots = [(slot, by_key[slot[-1]][level]) for slot in cur
                 if len(by_key.get(slot[-1], ())) > level and by_key[slot[-1]][level].op != "identity"]
        outs = _run([(cur[s].values, t) for s, t in slots])
        for (s, _), v in zip(slots, outs):
            cur[s] = JaggedTensor(v, cur[s].offsets, validate=False)
    new_kjts = {k: cur[("k", k)] for k in kjts}
    new_ikjts = [IKJT(ik.batch_size, ik.group_keys, ik.inverse_lookup,
                      {k: cur[("i", i, k)] for k in ik.per_feature}, validate=False)
                 for i, ik in enumerate(ikjts)]
    return new_kjts, new_ikjts
