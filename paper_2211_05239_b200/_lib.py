"""ctypes binding of librecd.so (the C ABI declared in include/recd.h).

The library is the product; this module only marshals torch CUDA tensors into
raw device pointers and the current CUDA stream.  There is no CPU fallback:
if the shared library is missing or the tensors are not on a CUDA device,
every op raises.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import torch

_LIB_PATH = Path(os.environ.get("RECD_LIB", Path(__file__).resolve().parent / "librecd.so"))
_lib = None

RECD_OK = 0
RECD_NO_ERROR = 0x7F7F7F7F7F7F7F7F
POOL_MODES = {"sum": 0, "avg": 1, "mean": 1, "max": 2}
POOL_SHARE = 0x100  # recd_pool_fwd mode flag (include/recd.h)
BWD_INVERSE, BWD_OCCURRENCES, BWD_GRAD, BWD_SCATTER = 1, 2, 4, 8  # recd_pool_bwd_stages
BWD_SETUP, BWD_SETUP_DONE = 16, 32  # bookkeeping alone / INVERSE without it
_ERRORS = {1: "invalid argument", 2: "CUDA error", 3: "scratch buffer too small",
           4: "unsupported configuration"}

_vp = C.c_void_p
_i32 = C.c_int32
_i64 = C.c_int64
_sz = C.c_size_t
_f32 = C.c_float
_pp = C.POINTER(C.c_void_p)
_p64 = C.POINTER(C.c_int64)
_p32 = C.POINTER(C.c_int32)

_SIGS = {
    "recd_version": (_i32, []),
    "recd_last_error": (C.c_char_p, []),
    "recd_launch_count": (_i64, []),
    "recd_debug_set_hash_mask": (None, [C.c_uint64]),
    "recd_debug_kernel_events": (None, [C.c_char_p, _vp, _vp]),
    "recd_dedup_scratch_bytes": (_sz, [_i32, _i32, _i64]),
    "recd_dedup": (_i32, [_i32, _p32, _i64, _pp, _pp, _p64, _pp, _pp, _pp, _vp, _vp, _sz, _vp]),
    "recd_dedup_number": (_i32, [_i32, _p32, _i64, _pp, _pp, _p64, _pp, _pp, _pp, _vp, _vp, _sz, _vp]),
    "recd_dedup_copy": (_i32, [_i32, _p32, _i64, _pp, _pp, _p64, _pp, _pp, _pp, _vp, _pp, _pp, _vp, _sz,
                               _vp]),
    "recd_dedup_ex": (_i32, [_i32, _p32, _i64, _pp, _pp, _p64, _vp, _i32, _pp, _pp, _pp, _vp, _pp,
                             _pp, _vp, _sz, _vp]),
    "recd_pool_fwd": (_i32, [_i32, _i64, _i32, _i32, _pp, _p64, _pp, _pp, _vp, _pp, _pp, _pp,
                             _vp, _vp]),
    "recd_pool_fwd_scatter": (_i32, [_i32, _i64, _i32, _i32, _pp, _p64, _pp, _pp, _vp, _i32, _pp, _pp,
                                     _vp, _vp]),
    "recd_expand": (_i32, [_i32, _i64, _i32, _pp, _pp, _pp, _vp]),
    "recd_embedding_lookup": (_i32, [_vp, _i64, _i32, _vp, _i64, _vp, _vp, _vp]),
    "recd_pool_dense": (_i32, [_vp, _i64, _i32, _vp, _i64, _i32, _vp, _vp]),
    "recd_pool_bwd_scratch_bytes": (_sz, [_i32, _i64, _i32, _p64]),
    "recd_pool_bwd": (_i32, [_i32, _i64, _i32, _i32, _pp, _p64, _pp, _pp, _p64, _vp, _pp, _pp,
                             _f32, _i32, _pp, _pp, _vp, _vp, _sz, _vp]),
    "recd_pool_bwd_prepare": (_i32, [_i32, _i64, _i32, _i32, _pp, _p64, _pp, _pp, _p64, _vp, _pp,
                                     _pp, _f32, _i32, _pp, _pp, _vp, _vp, _sz, _vp]),
    "recd_pool_bwd_finish": (_i32, [_i32, _i64, _i32, _i32, _pp, _p64, _pp, _pp, _p64, _vp, _pp,
                                    _pp, _f32, _i32, _pp, _pp, _vp, _vp, _sz, _vp]),
    "recd_rowcode_scratch_bytes": (_sz, [_i32, _i64]),
    "recd_rowcode_decode": (_i32, [_i32, _i64, _pp, _pp, _vp, _p64, _pp, _pp, _vp, _sz, _vp]),
    "recd_pool_bwd_csr": (_i32, [_i32, _i64, _i32, _i32, _pp, _p64, _pp, _pp, _p64, _vp, _pp, _pp,
                                 _f32, _i32, _pp, _pp, _vp, _vp, _sz, _pp, _pp]),
    "recd_pool_fwd_csr": (_i32, [_i32, _i64, _i32, _i32, _pp, _p64, _pp, _pp, _vp, _pp, _pp, _pp,
                                 _pp, _vp, _vp]),
    "recd_pool_bwd_stages": (_i32, [_i32, _i32, _i64, _i32, _i32, _pp, _p64, _pp, _pp, _p64, _vp,
                                    _pp, _pp, _f32, _i32, _pp, _pp, _vp, _vp, _sz, _vp]),
    "recd_wire_bound": (_i64, [_i32, C.POINTER(C.c_char_p), _i64, _i32, _p64, _p64]),
    "recd_wire_serialize": (_i32, [_i32, C.POINTER(C.c_char_p), _i64, _vp, _pp, _pp, _pp, _pp, _p64,
                                   _p64, _vp, _i64, _vp, _vp, _sz, _vp]),
    "recd_sort_pairs_scratch_bytes": (_sz, [_i32, _p64, _p64]),
    "recd_sort_pairs": (_i32, [_i32, _p64, _p64, _pp, _i32, _vp, _vp, _vp, _vp, _p32, _vp, _sz, _vp]),
    "recd_transform": (_i32, [_i32, _pp, _pp, _p64, _pp, _p32, _p64, _vp]),
    "recd_attention_pool_scratch_bytes": (_sz, [_i32, _i32, _p64]),
    "recd_attention_pool": (_i32, [_i32, _i64, _i32, _pp, _p64, _pp, _pp, _p64, _vp, _vp, _vp, _vp,
                                   _vp, _vp, _sz, _vp]),
    "recd_gemm_bf16_tn": (_i32, [_i32, _i32, _vp, _vp, _vp, _vp, _vp]),
    "recd_grad_unique_scratch_bytes": (_sz, [_i32, _i64]),
    "recd_grad_unique": (_i32, [_i32, _i64, _i32, _i32, _pp, _vp, _pp, _pp, _pp, _vp, _sz, _vp]),
    "recd_grad_unique_scatter": (_i32, [_i32, _i64, _i32, _i32, _pp, _vp, _pp, _pp, _i32, _pp, _pp, _vp,
                                        _sz, _vp]),
    "recd_sparse_sgd_scratch_bytes": (_sz, [_i32, _p64]),
    "recd_sparse_sgd": (_i32, [_i32, _i64, _i32, _pp, _p64, _pp, _pp, _p64, _vp, _pp, _f32, _i32,
                               _pp, _pp, _vp, _vp, _sz, _vp]),
    "recd_sparse_sgd_prepare": (_i32, [_i32, _i64, _i32, _pp, _p64, _pp, _pp, _p64, _vp, _pp, _f32, _i32,
                               _pp, _pp, _vp, _vp, _sz, _vp]),
    "recd_sparse_sgd_finish": (_i32, [_i32, _i64, _i32, _pp, _p64, _pp, _pp, _p64, _vp, _pp, _f32, _i32,
                               _pp, _pp, _vp, _vp, _sz, _vp]),
    "recd_shard_count_scratch_bytes": (_sz, [_i32, _i32, _i64]),
    "recd_shard_count": (_i32, [_i32, _i32, _i64, _pp, _pp, _vp, _pp, _vp, _vp, _sz, _vp]),
    "recd_shard_dispatch": (_i32, [_i32, _i32, _i64, _pp, _pp, _vp, _pp, _vp, _vp, _vp, _pp, _pp,
                                   _vp]),
    "recd_shard_scratch_bytes": (_sz, [_i32, _i32, _i64]),
    "recd_shard_bucketize": (_i32, [_i32, _i32, _i64, _pp, _pp, _vp, _pp, _pp, _vp, _vp, _sz,
                                    _vp]),
    "recd_shard_combine": (_i32, [_i32, _i32, _i64, _i32, _i32, _pp, _pp, _vp, _pp, _vp]),
    "recd_peer_ctl_words": (_i64, [_i32, _i32, _i32]),
    "recd_peer_alloc": (_i32, [_sz, _pp]),
    "recd_peer_free": (_i32, [_vp]),
    "recd_peer_export": (_i32, [_vp, _vp]),
    "recd_peer_import": (_i32, [_vp, _pp]),
    "recd_peer_close": (_i32, [_vp]),
    "recd_peer_exchange": (_i32, [_i32, _i32, _i32, _i32, _i32, _p32, _pp, _vp, _vp, _i64, _vp]),
    "recd_peer_copy_rows": (_i32, [_i32, _vp, _vp, _i32, _i64, _vp]),
    "recd_batched_copy_desc_bytes": (_sz, [_i32]),
    "recd_batched_copy": (_i32, [_i32, _pp, _pp, _p64, _vp, _vp, _vp]),
    "recd_exclusive_scan_scratch_bytes": (_sz, [_i32, _p64]),
    "recd_exclusive_scan": (_i32, [_i32, _pp, _pp, _p64, _vp, _vp, _vp, _sz, _vp]),
    "recd_jagged_scratch_bytes": (_sz, [_i32, _i64]),
    "recd_jagged_index_select_plan": (_i32, [_i32, _pp, _i64, _p64, _vp, _i64, _pp, _vp, _vp,
                                             _vp, _sz, _vp]),
    "recd_jagged_index_select_copy": (_i32, [_i32, _pp, _pp, _i64, _p64, _vp, _i64, _pp, _pp,
                                             _vp]),
    "recd_slice_scratch_bytes": (_sz, [_i64, _i64]),
    "recd_slice_renumber": (_i32, [_vp, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _sz, _vp]),
    "recd_partial_ikjt_scratch_bytes": (_sz, [_i64, _i64]),
    "recd_partial_ikjt": (_i32, [_i64, _i64, _vp, _vp, _i64, _vp, _vp, _vp, _p64, _p64, _vp, _sz, _vp]),
}

EXPORTS = tuple(_SIGS)


def lib_path() -> Path:
    return _LIB_PATH


def load(path: str | os.PathLike | None = None):
    """Load librecd.so (raises if it was not built -- no fallback)."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else _LIB_PATH
    if not p.exists():
        raise RuntimeError(
            f"{p} is missing: build the CUDA extension with "
            "`python -m paper_2211_05239_b200.build` (there is no CPU fallback)")
    lib = C.CDLL(str(p))
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib


def check(rc: int, what: str) -> None:
    if rc != RECD_OK:
        detail = load().recd_last_error().decode() or _ERRORS.get(rc, "")
        raise RuntimeError(f"{what} failed: {_ERRORS.get(rc, rc)} {detail}".strip())


def require_cuda(*tensors: torch.Tensor) -> None:
    for t in tensors:
        if t is not None and not t.is_cuda:
            raise ValueError("the IKJT hot path runs on CUDA tensors only (no CPU fallback)")


def ptrs(ts) -> C.Array:
    arr = (C.c_void_p * max(1, len(ts)))()
    for i, t in enumerate(ts):
        arr[i] = None if t is None else (t if isinstance(t, int) else t.data_ptr())
    return arr


def i64s(xs) -> C.Array:
    arr = (C.c_int64 * max(1, len(xs)))()
    for i, x in enumerate(xs):
        arr[i] = int(x)
    return arr


def i32s(xs) -> C.Array:
    arr = (C.c_int32 * max(1, len(xs)))()
    for i, x in enumerate(xs):
        arr[i] = int(x)
    return arr


def stream_ptr(device: torch.device | None = None) -> int:
    return torch.cuda.current_stream(device).cuda_stream


class Workspace:
    """Grow-only device scratch arena per device (the C ABI never allocates)."""

    _bufs: dict = {}

    @classmethod
    def get(cls, nbytes: int, device: torch.device, tag: str = "default") -> torch.Tensor:
        key = (str(device), tag)
        buf = cls._bufs.get(key)
        if buf is None or buf.numel() < nbytes:
            buf = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)
            cls._bufs[key] = buf
        return buf


def launch_count() -> int:
    return int(load().recd_launch_count())


def set_hash_mask(mask: int) -> None:
    """Test hook: weaken the row hash to force collisions (0 or ~0 restores)."""
    load().recd_debug_set_hash_mask(C.c_uint64(mask & 0xFFFFFFFFFFFFFFFF))
