"""Jagged / keyed-jagged / inverse-keyed-jagged tensors on B200.

Drop-in for `sessiondedup.tensors` (/root/reference/pkg/src/sessiondedup/
tensors.py): same type names, fields, invariants, error messages and first-
occurrence semantics, but the buffers are int64 CUDA tensors and every
conversion runs in librecd's sm_100a kernels:

  build_kjt(rows, keys)        tensors.py:246-254  (host packing + one H2D copy)
  build_ikjt(rows, group)      tensors.py:269-308  -> recd_dedup
  kjt_to_ikjts(kjt, groups)    reader.convert's per-group loop (reader.py:166),
                               all groups deduplicated in one recd_dedup call
  ikjt_to_kjt(ikjt)            tensors.py:393-399  -> recd_jagged_index_select_*
  jagged_index_select(jt, idx) tensors.py:363-390  -> recd_jagged_index_select_*
  slice_ikjt_rows / split_ikjt trainer_sim.py:394-446 -> recd_slice_renumber
  build_partial_ikjt(rows, key) tensors.py:311-360  -> recd_dedup + recd_partial_ikjt
"""

from __future__ import annotations

from typing import Iterable, Mapping, Sequence

import ctypes

import numpy as np
import torch

from . import _lib

__all__ = [
    "JaggedTensor",
    "KJT",
    "IKJT",
    "build_kjt",
    "build_ikjt",
    "kjt_to_ikjt",
    "kjt_to_ikjts",
    "ikjt_to_kjt",
    "jagged_index_select",
    "slice_ikjt_rows",
    "split_ikjt",
    "PartialIKJT",
    "build_partial_ikjt",
    "kjt_to_partial_ikjt",
    "jt_equal",
    "kjt_equal",
    "default_device",
]


def default_device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device: the IKJT hot path has no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def _as_ids(x, device) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        t = x.to(device=device, dtype=torch.int64)
    else:
        t = torch.as_tensor(np.asarray(x, dtype=np.int64), device=device)
    if t.dim() != 1:
        raise ValueError(f"ID list must be one-dimensional, got shape {tuple(t.shape)}")
    return t.contiguous()


class JaggedTensor:
    """int64 values + one offset per row; the last row runs to len(values)
    (tensors.py:60-111).  Validation matches the reference's __post_init__."""

    __slots__ = ("values", "offsets")

    def __init__(self, values, offsets, *, device=None, validate: bool = True):
        dev = device or (values.device if isinstance(values, torch.Tensor) and values.is_cuda
                         else default_device())
        object.__setattr__(self, "values", _as_ids(values, dev))
        object.__setattr__(self, "offsets", _as_ids(offsets, dev))
        if validate and self.offsets.numel():
            off = self.offsets
            if int(off[0]) != 0:
                raise ValueError("offsets[0] must be 0")
            if off.numel() > 1 and bool((off[1:] < off[:-1]).any()):
                raise ValueError("offsets must be non-decreasing")
            if int(off[-1]) > self.values.numel():
                raise ValueError("offset exceeds values length")

    def __setattr__(self, name, value):
        raise AttributeError("JaggedTensor is immutable")

    @classmethod
    def _trusted(cls, values: torch.Tensor, offsets: torch.Tensor) -> "JaggedTensor":
        jt = object.__new__(cls)
        object.__setattr__(jt, "values", values)
        object.__setattr__(jt, "offsets", offsets)
        return jt

    @classmethod
    def from_rows(cls, rows: Sequence, device=None) -> "JaggedTensor":
        """tensors.py:84-92."""
        v, o = _pack_rows([np.asarray(r, dtype=np.int64).reshape(-1) for r in rows])
        dev = device or default_device()
        return cls._trusted(torch.from_numpy(v).to(dev), torch.from_numpy(o).to(dev))

    @property
    def device(self) -> torch.device:
        return self.values.device

    @property
    def row_count(self) -> int:
        return int(self.offsets.numel())

    def row_lengths(self) -> torch.Tensor:
        bounds = torch.cat([self.offsets, self.offsets.new_tensor([self.values.numel()])])
        return bounds[1:] - bounds[:-1]

    def row(self, i: int) -> torch.Tensor:
        n = self.row_count
        if not 0 <= i < n:
            raise IndexError(f"row {i} out of range for {n} rows")
        start = int(self.offsets[i])
        end = int(self.offsets[i + 1]) if i + 1 < n else self.values.numel()
        return self.values[start:end]

    def to_pylists(self) -> list[list[int]]:
        v = self.values.cpu().numpy()
        o = self.offsets.cpu().numpy()
        ends = np.append(o[1:], v.size) if o.size else o
        return [v[s:e].tolist() for s, e in zip(o, ends)]

    def numpy(self) -> tuple[np.ndarray, np.ndarray]:
        return self.values.cpu().numpy(), self.offsets.cpu().numpy()


def jt_equal(a: JaggedTensor, b: JaggedTensor) -> bool:
    return torch.equal(a.values, b.values) and torch.equal(a.offsets, b.offsets)


class KJT:
    """One JaggedTensor of batch_size rows per key (tensors.py:118-137)."""

    def __init__(self, batch_size: int, entries: Mapping[str, JaggedTensor]):
        if batch_size < 1:
            raise ValueError("batch_size must be >= 1")
        self.batch_size = int(batch_size)
        self.entries = dict(entries)
        for key, jt in self.entries.items():
            if jt.row_count != self.batch_size:
                raise ValueError(f"feature {key!r} has {jt.row_count} rows, expected {self.batch_size}")

    @property
    def keys(self) -> tuple[str, ...]:
        return tuple(self.entries)


def kjt_equal(a: KJT, b: KJT) -> bool:
    if a.batch_size != b.batch_size or a.keys != b.keys:
        return False
    return all(jt_equal(a.entries[k], b.entries[k]) for k in a.entries)


class IKJT:
    """Deduplicated encoding of one feature group (tensors.py:146-191):
    inverse_lookup[i] is the unique-row ordinal of batch row i; every
    per-feature JaggedTensor has U rows in first-occurrence order."""

    def __init__(self, batch_size: int, group_keys: Sequence[str], inverse_lookup,
                 per_feature: Mapping[str, JaggedTensor], *, validate: bool = True):
        self.batch_size = int(batch_size)
        self.group_keys = tuple(group_keys)
        dev = next(iter(per_feature.values())).device if per_feature else default_device()
        self.inverse_lookup = _as_ids(inverse_lookup, dev)
        self.per_feature = dict(per_feature)
        if not validate:
            return
        if self.batch_size < 1:
            raise ValueError("batch_size must be >= 1")
        if self.inverse_lookup.numel() != self.batch_size:
            raise ValueError("inverse_lookup must have one entry per batch row")
        if set(self.group_keys) != set(self.per_feature):
            raise ValueError("group_keys and per_feature keys differ")
        u = self.unique_count
        if u > self.batch_size:
            raise ValueError("more unique rows than batch rows")
        for key, jt in self.per_feature.items():
            if jt.row_count != u:
                raise ValueError(f"feature {key!r} has {jt.row_count} dedup rows, expected {u}")
        if self.inverse_lookup.numel():
            lo = int(self.inverse_lookup.min())
            hi = int(self.inverse_lookup.max())
            if lo < 0 or hi >= u:
                raise ValueError("inverse_lookup entry out of range")
            if torch.unique(self.inverse_lookup).numel() != u:
                raise ValueError("orphan unique rows: some ordinal never referenced")

    @property
    def unique_count(self) -> int:
        return self.per_feature[self.group_keys[0]].row_count

    @property
    def device(self) -> torch.device:
        return self.inverse_lookup.device


# ----------------------------------------------------------------- host side
def _row_features(row) -> Mapping:
    feats = getattr(row, "features", None)
    if feats is not None:
        return feats
    if isinstance(row, Mapping):
        return row
    raise TypeError(f"cannot extract features from {type(row).__name__}")


def _feature_list(row, key: str) -> np.ndarray:
    seq = _row_features(row).get(key)
    if seq is None:
        return np.empty(0, dtype=np.int64)  # absent keys are empty lists (tensors.py:237-243)
    arr = np.asarray(seq, dtype=np.int64)
    if arr.ndim != 1:
        raise ValueError(f"ID list must be one-dimensional, got shape {arr.shape}")
    return arr


def _pack_rows(arrs: Sequence[np.ndarray]) -> tuple[np.ndarray, np.ndarray]:
    lengths = np.fromiter((a.size for a in arrs), dtype=np.int64, count=len(arrs))
    offsets = np.zeros(len(arrs), dtype=np.int64)
    if len(arrs) > 1:
        np.cumsum(lengths[:-1], out=offsets[1:])
    values = np.concatenate(arrs).astype(np.int64, copy=False) if arrs else np.empty(0, np.int64)
    return values, offsets


def _as_id_array(seq) -> np.ndarray:
    """tensors.py:47-51: the conversion the native packer falls back to for
    ID lists that are not plain Python ints (floats, numpy arrays, scalars)."""
    arr = np.asarray(seq, dtype=np.int64)
    if arr.ndim != 1:
        raise ValueError(f"ID list must be one-dimensional, got shape {arr.shape}")
    return np.ascontiguousarray(arr)


def build_kjt(rows: Sequence, keys: Sequence[str], device=None) -> KJT:
    """Records -> KJT on the GPU, preserving batch order (tensors.py:246-254).
    The records are walked once in native code (`_hostpack.pack_rows`,
    csrc/host/recd_hostpack.cpp) instead of one np.asarray per list."""
    if len(rows) == 0:
        raise ValueError("empty batch")
    from . import _hostpack  # built by build.build_host(); no Python fallback
    dev = device or default_device()
    packed = _hostpack.pack_rows(rows, list(keys), _as_id_array)
    entries = {}
    for key, (vb, ob) in zip(keys, packed):
        v = torch.frombuffer(bytearray(vb), dtype=torch.int64) if vb else torch.empty(0, dtype=torch.int64)
        o = torch.frombuffer(bytearray(ob), dtype=torch.int64)
        entries[key] = JaggedTensor._trusted(v.to(dev, non_blocking=True), o.to(dev, non_blocking=True))
    return KJT(len(rows), entries)


# ---------------------------------------------------------------- dedup
def kjt_to_ikjts(kjt: KJT, groups: Sequence[Sequence[str]]) -> list[IKJT]:
    """Deduplicate every group of a KJT in ONE batched recd_dedup call.

    Semantics per group are exactly build_ikjt's (tensors.py:269-308)."""
    groups = [tuple(g) for g in groups]
    if any(len(g) == 0 for g in groups):
        raise ValueError("empty dedup group")
    if not groups:
        return []
    lib = _lib.load()
    B = kjt.batch_size
    feats = [kjt.entries[k] for g in groups for k in g]
    dev = feats[0].device
    _lib.require_cuda(*[f.values for f in feats])
    F = len(feats)
    inverse = [torch.empty(B, dtype=torch.int64, device=dev) for _ in groups]
    uoff = [torch.empty(B, dtype=torch.int64, device=dev) for _ in feats]
    uval = [torch.empty(max(f.values.numel(), 1), dtype=torch.int64, device=dev) for f in feats]
    counts = torch.empty(2 * F, dtype=torch.int64, device=dev)
    nbytes = lib.recd_dedup_scratch_bytes(len(groups), F, B)
    scratch = _lib.Workspace.get(nbytes, dev, "dedup")
    rc = lib.recd_dedup(len(groups), _lib.i32s([len(g) for g in groups]), B,
                        _lib.ptrs([f.values for f in feats]), _lib.ptrs([f.offsets for f in feats]),
                        _lib.i64s([f.values.numel() for f in feats]), _lib.ptrs(inverse),
                        _lib.ptrs(uoff), _lib.ptrs(uval), counts.data_ptr(), scratch.data_ptr(),
                        scratch.numel(), _lib.stream_ptr(dev))
    _lib.check(rc, "recd_dedup")
    c = counts.cpu().tolist()
    out, f = [], 0
    for gi, g in enumerate(groups):
        per = {}
        for key in g:
            per[key] = JaggedTensor._trusted(uval[f][: c[F + f]], uoff[f][: c[f]])
            f += 1
        out.append(IKJT(B, g, inverse[gi], per, validate=False))
    return out


def kjt_to_ikjt(kjt: KJT, group: Sequence[str]) -> IKJT:
    if len(group) == 0:
        raise ValueError("empty dedup group")
    return kjt_to_ikjts(kjt, [group])[0]


def build_ikjt(rows: Sequence, group: Sequence[str], device=None) -> IKJT:
    """tensors.py:269-308: rows i, j share an inverse entry iff all features
    in the group have identical lists; unique rows in first-occurrence order."""
    if len(rows) == 0:
        raise ValueError("empty batch")
    if len(group) == 0:
        raise ValueError("empty dedup group")
    return kjt_to_ikjt(build_kjt(rows, group, device), group)


# ------------------------------------------------------- jagged index select
def _select(jts: Sequence[JaggedTensor], idx: torch.Tensor) -> list[JaggedTensor]:
    lib = _lib.load()
    dev = jts[0].device
    nrows = jts[0].row_count
    n = idx.numel()
    F = len(jts)
    out_off = [torch.empty(max(n, 1), dtype=torch.int64, device=dev) for _ in jts]
    totals = torch.empty(F, dtype=torch.int64, device=dev)
    err = torch.empty(1, dtype=torch.int64, device=dev)
    scratch = _lib.Workspace.get(lib.recd_jagged_scratch_bytes(F, n), dev, "jagged")
    nv = _lib.i64s([j.values.numel() for j in jts])
    rc = lib.recd_jagged_index_select_plan(F, _lib.ptrs([j.offsets for j in jts]), nrows, nv,
                                           idx.data_ptr(), n, _lib.ptrs(out_off),
                                           totals.data_ptr(), err.data_ptr(), scratch.data_ptr(),
                                           scratch.numel(), _lib.stream_ptr(dev))
    _lib.check(rc, "recd_jagged_index_select_plan")
    host = torch.cat([err, totals]).cpu().tolist()
    if host[0] != _lib.RECD_NO_ERROR:
        p = host[0]
        raise IndexError(f"index {int(idx[p])} at position {p} out of range for {nrows} rows")
    out_val = [torch.empty(max(t, 1), dtype=torch.int64, device=dev) for t in host[1:]]
    rc = lib.recd_jagged_index_select_copy(F, _lib.ptrs([j.values for j in jts]),
                                           _lib.ptrs([j.offsets for j in jts]), nrows, nv,
                                           idx.data_ptr(), n, _lib.ptrs(out_off),
                                           _lib.ptrs(out_val), _lib.stream_ptr(dev))
    _lib.check(rc, "recd_jagged_index_select_copy")
    return [JaggedTensor._trusted(v[:t], o[:n]) for v, o, t in zip(out_val, out_off, host[1:])]


def jagged_index_select(jt: JaggedTensor, indices) -> JaggedTensor:
    """Output row k equals input row indices[k] (tensors.py:363-390)."""
    idx = _as_ids(indices, jt.device)
    return _select([jt], idx)[0]


def ikjt_to_kjt(ikjt: IKJT) -> KJT:
    """Expand an IKJT back to the logically equal KJT (tensors.py:393-399);
    all features of the group are expanded in one launch sequence."""
    keys = list(ikjt.per_feature)
    outs = _select([ikjt.per_feature[k] for k in keys], ikjt.inverse_lookup)
    return KJT(ikjt.batch_size, dict(zip(keys, outs)))


# ------------------------------------------------------------- DP slicing
def slice_ikjt_rows(ikjt: IKJT, start: int, stop: int) -> IKJT:
    """Rows [start, stop) without re-hashing; surviving unique rows are
    renumbered in first-occurrence order (trainer_sim.py:394-413)."""
    if not 0 <= start < stop <= ikjt.batch_size:
        raise ValueError(f"bad row range [{start}, {stop})")
    lib = _lib.load()
    dev = ikjt.device
    n = stop - start
    U = ikjt.unique_count
    new_inv = torch.empty(n, dtype=torch.int64, device=dev)
    order = torch.empty(n, dtype=torch.int64, device=dev)
    count = torch.empty(1, dtype=torch.int64, device=dev)
    scratch = _lib.Workspace.get(lib.recd_slice_scratch_bytes(U, n), dev, "slice")
    rc = lib.recd_slice_renumber(ikjt.inverse_lookup.data_ptr(), start, stop, U,
                                 new_inv.data_ptr(), order.data_ptr(), count.data_ptr(),
                                 scratch.data_ptr(), scratch.numel(), _lib.stream_ptr(dev))
    _lib.check(rc, "recd_slice_renumber")
    k = int(count.item())
    keys = list(ikjt.per_feature)
    outs = _select([ikjt.per_feature[key] for key in keys], order[:k])
    return IKJT(n, ikjt.group_keys, new_inv, dict(zip(keys, outs)), validate=False)


def split_ikjt(ikjt: IKJT, num_ranks: int) -> list[IKJT]:
    """Contiguous per-rank chunks, first B mod R take one extra row
    (split_batch, trainer_sim.py:416-446)."""
    if num_ranks < 1:
        raise ValueError("num_ranks must be >= 1")
    if ikjt.batch_size < num_ranks:
        raise ValueError(f"cannot split {ikjt.batch_size} rows across {num_ranks} ranks")
    base, extra = divmod(ikjt.batch_size, num_ranks)
    out, start = [], 0
    for r in range(num_ranks):
        stop = start + base + (1 if r < extra else 0)
        out.append(slice_ikjt_rows(ikjt, start, stop))
        start = stop
    return out


# --------------------------------------------------------- partial IKJT
class PartialIKJT:
    """Single-feature shift-aware encoding (tensors.py:194-225): rows are
    (offset, length) windows into one shared value buffer."""

    def __init__(self, feature_key: str, values, windows, *, validate: bool = True):
        dev = values.device if isinstance(values, torch.Tensor) and values.is_cuda else default_device()
        self.feature_key = feature_key
        self.values = _as_ids(values, dev)
        w = windows if isinstance(windows, torch.Tensor) else torch.as_tensor(
            np.asarray(windows, dtype=np.int64))
        self.windows = w.to(device=dev, dtype=torch.int64).contiguous()
        if not validate:
            return
        if self.windows.dim() != 2 or self.windows.shape[1] != 2:
            raise ValueError("windows must be a (B, 2) array")
        if self.windows.numel():
            if bool((self.windows[:, 0] + self.windows[:, 1] > self.values.numel()).any()):
                raise ValueError("window exceeds value buffer")
            if bool((self.windows < 0).any()):
                raise ValueError("negative window bound")

    @property
    def row_count(self) -> int:
        return int(self.windows.shape[0])

    def row(self, i: int) -> torch.Tensor:
        off, length = (int(x) for x in self.windows[i].tolist())
        return self.values[off:off + length]


def kjt_to_partial_ikjt(kjt: KJT, key: str, ikjt: IKJT | None = None) -> PartialIKJT:
    """build_partial_ikjt on a KJT already on the GPU (recd_dedup of the key,
    then recd_partial_ikjt over its unique rows).  `ikjt` may pass an existing
    exact dedup of the key to skip the first step."""
    if ikjt is None:
        ikjt = kjt_to_ikjt(kjt, [key])
    lib = _lib.load()
    jt = ikjt.per_feature[key]
    dev = jt.device
    B, U, nval = ikjt.batch_size, jt.row_count, int(jt.values.numel())
    values = torch.empty(max(nval, 1), dtype=torch.int64, device=dev)
    windows = torch.empty((B, 2), dtype=torch.int64, device=dev)
    scratch = _lib.Workspace.get(lib.recd_partial_ikjt_scratch_bytes(U, nval), dev, "partial")
    n_out, rounds = ctypes.c_int64(0), ctypes.c_int64(0)
    rc = lib.recd_partial_ikjt(B, U, jt.values.data_ptr(), jt.offsets.data_ptr(), nval,
                               ikjt.inverse_lookup.data_ptr(), values.data_ptr(), windows.data_ptr(),
                               ctypes.byref(n_out), ctypes.byref(rounds), scratch.data_ptr(),
                               scratch.numel(), _lib.stream_ptr(dev))
    _lib.check(rc, "recd_partial_ikjt")
    out = PartialIKJT(key, values[: n_out.value], windows, validate=False)
    out.rounds = int(rounds.value)
    return out


def build_partial_ikjt(rows: Sequence, key: str, device=None) -> PartialIKJT:
    """tensors.py:311-338: greedy batch-order shift-aware encoding of one
    feature -- reuse the leftmost window equal to the row, else append the
    row minus its longest prefix matching the buffer's suffix."""
    if len(rows) == 0:
        raise ValueError("empty batch")
    return kjt_to_partial_ikjt(build_kjt(rows, [key], device), key)
