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

import time
from dataclasses import dataclass, field, replace
from typing import Mapping, Sequence

import numpy as np
import torch

from . import _lib
from .tensors import IKJT, KJT, JaggedTensor, build_kjt, kjt_to_ikjts

__all__ = ["Transform", "apply_transform", "DataloaderSpec", "ReaderBatch", "StageTimings",
           "convert", "process", "process_tensors"]

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


def process_tensors(kjts: Mapping[str, JaggedTensor], ikjts: Sequence[IKJT],
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


@dataclass(frozen=True)
class DataloaderSpec:
    """reader.DataloaderSpec (reader.py:86-121): keys, dedup groups, transforms."""

    keys: tuple[str, ...]
    dedup_sparse_features: tuple[tuple[str, ...], ...]
    transforms: tuple[Transform, ...] = ()
    batch_size: int = 4096

    def __post_init__(self) -> None:
        if self.batch_size < 1:
            raise ValueError("batch_size must be >= 1")
        seen: set[str] = set()
        for group in self.dedup_sparse_features:
            if not group:
                raise ValueError("empty dedup group")
            for key in group:
                if key in seen:
                    raise ValueError(f"feature {key!r} in more than one dedup group")
                if key not in self.keys:
                    raise ValueError(f"grouped feature {key!r} not in keys")
                seen.add(key)
        for t in self.transforms:
            if t.key not in self.keys:
                raise ValueError(f"transform targets unknown key {t.key!r}")

    @property
    def plain_keys(self) -> tuple[str, ...]:
        grouped = {k for g in self.dedup_sparse_features for k in g}
        return tuple(k for k in self.keys if k not in grouped)

    def without_dedup(self) -> "DataloaderSpec":
        """The baseline spec: same keys and transforms, no dedup groups."""
        return replace(self, dedup_sparse_features=())


@dataclass
class StageTimings:
    fill_s: float = 0.0
    convert_s: float = 0.0
    process_s: float = 0.0

    @property
    def total_s(self) -> float:
        return self.fill_s + self.convert_s + self.process_s


@dataclass
class ReaderBatch:
    """reader.ReaderBatch (reader.py:136-150) on device tensors."""

    batch_size: int
    kjts: dict[str, JaggedTensor]
    ikjts: list[IKJT]
    labels: np.ndarray
    stage_timings: StageTimings = field(default_factory=StageTimings)
    bytes_in: int = 0
    bytes_out: int = 0

    def all_keys(self) -> tuple[str, ...]:
        keys = list(self.kjts)
        for ikjt in self.ikjts:
            keys.extend(ikjt.group_keys)
        return tuple(keys)


def convert(rows, spec: DataloaderSpec) -> ReaderBatch:
    """reader.convert (reader.py:160-175): one IKJT per dedup group, one plain
    jagged tensor per remaining key.  The records are packed once in native
    code (all keys), copied to the GPU, and every group is deduplicated in one
    batched recd_dedup."""
    if not rows:
        raise ValueError("convert needs a non-empty row batch")
    t0 = time.perf_counter()
    keys = list(spec.keys)
    kjt = build_kjt(rows, keys)
    groups = [list(g) for g in spec.dedup_sparse_features]
    ikjts = kjt_to_ikjts(kjt, groups) if groups else []
    kjts = {k: kjt.entries[k] for k in spec.plain_keys}
    labels = np.fromiter((r.label for r in rows), dtype=np.int64, count=len(rows))
    batch = ReaderBatch(batch_size=len(rows), kjts=kjts, ikjts=ikjts, labels=labels)
    torch.cuda.synchronize()
    batch.stage_timings.convert_s = time.perf_counter() - t0
    return batch


def process(batch: ReaderBatch, transforms: Sequence[Transform]) -> ReaderBatch:
    """reader.process (reader.py:178-217): element-wise transforms; IKJT features
    are transformed on their deduplicated values only and stay IKJTs."""
    t0 = time.perf_counter()
    kjts, ikjts = process_tensors(batch.kjts, batch.ikjts, transforms)
    out = ReaderBatch(batch_size=batch.batch_size, kjts=kjts, ikjts=ikjts, labels=batch.labels,
                      stage_timings=batch.stage_timings, bytes_in=batch.bytes_in,
                      bytes_out=batch.bytes_out)
    out.stage_timings.process_s += time.perf_counter() - t0
    return out
