"""B200-native IKJT training hot path (RecD, arXiv 2211.05239).

Drop-in for the hot path of the reference's `sessiondedup` package:
KJT -> IKJT dedup, deduplicated pooled embedding lookup with inverse
expansion, and its backward with a deterministic sorted scatter-add -- all in
hand-written sm_100a kernels behind the C ABI in `include/recd.h`
(`librecd.so`, loaded through ctypes; no CPU fallback).
"""

from .tensors import (  # noqa: F401
    IKJT,
    KJT,
    JaggedTensor,
    PartialIKJT,
    build_partial_ikjt,
    kjt_to_partial_ikjt,
    build_ikjt,
    build_kjt,
    ikjt_to_kjt,
    jagged_index_select,
    jt_equal,
    kjt_equal,
    kjt_to_ikjt,
    kjt_to_ikjts,
    slice_ikjt_rows,
    split_ikjt,
)
from .embedding import (  # noqa: F401
    ELEMENT_POOLING,
    DedupEmbeddingBagCollection,
    EmbeddingTable,
    embedding_lookup,
    pool,
    pooled_lookup,
    pooled_lookup_backward,
)
from .wire import serialize_ikjt, serialize_kjt, slice_stream_bytes, values_stream_bytes  # noqa: F401
from .encoder import DedupAttentionPool, attention_pool_macs  # noqa: F401
from ._lib import launch_count, lib_path, load as load_library  # noqa: F401

__version__ = "0.1.0"
