"""Canonical wire format of KJTs / IKJTs on the GPU (tensors.py:463-515).

`serialize_kjt` / `serialize_ikjt` return the same bytes as the reference's
functions; the stream is assembled on the device by `recd_wire_serialize`
(one launch pair, sizes read on the device) and copied to the host once.
`serialize_to_device` keeps it on the GPU (e.g. for an NVLink / network send)
and returns (buffer, device byte count).  `slice_stream_bytes` /
`values_stream_bytes` are the reference's byte-accounting helpers
(trainer_sim.py:281-305 counts the all-to-all with them).
"""

from __future__ import annotations

import ctypes as C
from typing import Mapping, Sequence

import torch

from . import _lib
from .tensors import IKJT, KJT, JaggedTensor

__all__ = ["serialize_kjt", "serialize_ikjt", "serialize_to_device", "slice_stream_bytes",
           "values_stream_bytes"]


def _names(keys: Sequence[str]):
    enc = [k.encode("utf-8") for k in keys]
    return (C.c_char_p * max(len(enc), 1))(*enc), enc


def serialize_to_device(keys: Sequence[str], batch_size: int, inverse: torch.Tensor | None,
                        tensors: Mapping[str, JaggedTensor]) -> tuple[torch.Tensor, torch.Tensor]:
    """(uint8 device buffer, int64 device byte count) holding `_serialize`'s bytes."""
    lib = _lib.load()
    keys = list(keys)
    feats = [tensors[k] for k in keys]
    dev = feats[0].device if feats else (inverse.device if inverse is not None else _lib_device())
    names, _ = _names(keys)
    ocaps = [f.offsets.numel() for f in feats]
    vcaps = [f.values.numel() for f in feats]
    bound = lib.recd_wire_bound(len(keys), names, int(batch_size), 1 if inverse is not None else 0,
                                _lib.i64s(ocaps), _lib.i64s(vcaps))
    if bound < 0:
        raise ValueError("too many keys for the wire format")
    out = torch.empty(max(int(bound), 8) + 8, dtype=torch.uint8, device=dev)
    total = torch.empty(1, dtype=torch.int64, device=dev)
    scratch = _lib.Workspace.get(4096, dev, "wire")
    rc = lib.recd_wire_serialize(len(keys), names, int(batch_size),
                                 inverse.data_ptr() if inverse is not None else None,
                                 _lib.ptrs([f.offsets for f in feats]), _lib.ptrs([f.values for f in feats]),
                                 None, None, _lib.i64s(ocaps), _lib.i64s(vcaps), out.data_ptr(), out.numel(),
                                 total.data_ptr(), scratch.data_ptr(), scratch.numel(), _lib.stream_ptr(dev))
    _lib.check(rc, "recd_wire_serialize")
    return out, total


def _lib_device():
    return torch.device("cuda", torch.cuda.current_device())


def _to_bytes(buf: torch.Tensor, total: torch.Tensor) -> bytes:
    n = int(total.item())
    if n < 0:
        raise RuntimeError("wire buffer too small")
    return bytes(buf[:n].cpu().numpy().tobytes())


def serialize_kjt(kjt: KJT) -> bytes:
    """tensors.serialize_kjt (tensors.py:497-498)."""
    return _to_bytes(*serialize_to_device(kjt.keys, kjt.batch_size, None, kjt.entries))


def serialize_ikjt(ikjt: IKJT) -> bytes:
    """tensors.serialize_ikjt (tensors.py:501-504)."""
    return _to_bytes(*serialize_to_device(ikjt.group_keys, ikjt.batch_size, ikjt.inverse_lookup,
                                          ikjt.per_feature))


def slice_stream_bytes(jt: JaggedTensor) -> int:
    """Wire size of one feature's (offsets, values) slices (tensors.py:507-510)."""
    return 16 + 8 * (jt.offsets.numel() + jt.values.numel())


def values_stream_bytes(jt: JaggedTensor) -> int:
    """Data bytes of the values stream alone (tensors.py:513-515)."""
    return 8 * jt.values.numel()
