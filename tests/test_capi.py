"""The C-ABI library loads (no GPU needed) and exports every declared symbol."""

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def _declared():
    text = (ROOT / "include" / "recd.h").read_text()
    return sorted(set(re.findall(r"\b(recd_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_hot_path():
    names = _declared()
    for n in ("recd_dedup", "recd_pool_fwd", "recd_pool_bwd", "recd_jagged_index_select_plan",
              "recd_jagged_index_select_copy", "recd_slice_renumber", "recd_embedding_lookup",
              "recd_pool_dense"):
        assert n in names


def test_library_exports_every_declared_symbol():
    from paper_2211_05239_b200 import _lib
    if not _lib.lib_path().exists():
        from paper_2211_05239_b200.build import build
        build()
    lib = ctypes.CDLL(str(_lib.lib_path()))
    for n in _declared():
        assert hasattr(lib, n), n
    # the ctypes signature table covers every declared entry point
    assert set(_declared()) == set(_lib.EXPORTS)


def test_host_library_exports_its_header():
    """librecd_host.so (the row-delta encoder of the H2D path) exports every
    function include/recd_host.h declares."""
    from paper_2211_05239_b200 import rowcode
    text = (ROOT / "include" / "recd_host.h").read_text()
    names = sorted(set(re.findall(r"\b(recd_[a-z0-9_]+)\s*\(", text)))
    assert names == ["recd_rowcode_encode"]
    lib = rowcode.load_host()
    for n in names:
        assert hasattr(lib, n), n


def test_host_only_entry_points_without_gpu():
    from paper_2211_05239_b200 import _lib
    lib = _lib.load()
    assert lib.recd_version() >= 1
    assert lib.recd_dedup_scratch_bytes(26, 26, 65536) > 0
    assert lib.recd_pool_bwd_scratch_bytes(2, 1024, 64, _lib.i64s([4096, 4096])) > 0
    assert lib.recd_jagged_scratch_bytes(1, 100) > 0
    # argument validation happens before any device work
    rc = lib.recd_dedup(0, None, 1, None, None, None, None, None, None, None, None, 0, None)
    assert rc == 1
    # partial IKJT: scratch grows with the unique values; bad sizes rejected up front
    assert lib.recd_partial_ikjt_scratch_bytes(65536, 1 << 20) > lib.recd_partial_ikjt_scratch_bytes(65536, 1)
    rc = lib.recd_partial_ikjt(4, 5, None, None, 0, None, None, None, None, None, None, 0, None)
    assert rc == 1


def test_no_cpu_fallback():
    import torch
    from paper_2211_05239_b200 import _lib
    with pytest.raises(ValueError, match="no CPU fallback"):
        _lib.require_cuda(torch.zeros(1))


def test_scratch_sizes_cover_every_backward_entry_point():
    """The scratch-size queries must cover what each entry point carves: with
    exactly the queried size the call gets past the scratch check (no GPU here,
    so it then fails launching: RECD_ERR_CUDA = 2, not RECD_ERR_SCRATCH = 3)."""
    import ctypes as C
    from paper_2211_05239_b200 import _lib
    lib = _lib.load()
    F, rows, D = 2, 3000, 8
    caps = _lib.i64s([500, 700])
    fake = [C.c_void_p(4096 * (i + 1)) for i in range(8)]
    P = lambda *xs: (C.c_void_p * len(xs))(*[x.value for x in xs])  # noqa: E731
    nb = lib.recd_sparse_sgd_scratch_bytes(F, caps)
    for fn in (lib.recd_sparse_sgd, lib.recd_sparse_sgd_prepare, lib.recd_sparse_sgd_finish):
        rc = fn(F, rows, D, P(fake[0], fake[1]), _lib.i64s([rows, rows]), P(fake[2], fake[3]),
                P(fake[4], fake[5]), caps, fake[6].value, P(fake[6], fake[7]), C.c_float(0.1), 1,
                None, None, None, fake[7].value, nb, None)
        assert rc != 3, rc
    B = 1024
    nb = lib.recd_pool_bwd_scratch_bytes(F, B, D, caps)
    stages = [lambda *a, st=st: lib.recd_pool_bwd_stages(st, *a) for st in (1, 2, 4, 8)]
    for fn in (lib.recd_pool_bwd, lib.recd_pool_bwd_prepare, lib.recd_pool_bwd_finish, *stages):
        rc = fn(F, B, D, 0, P(fake[0], fake[1]), _lib.i64s([rows, rows]), P(fake[2], fake[3]),
                P(fake[4], fake[5]), caps, fake[6].value, P(fake[6], fake[6]), P(fake[7], fake[7]),
                C.c_float(0.1), 1, None, None, None, fake[7].value, nb, None)
        assert rc != 3, rc


def test_pool_bwd_csr_points_into_scratch():
    """recd_pool_bwd_csr launches nothing: on the CPU it returns where the
    inverse CSR of each feature lives inside the backward scratch (features
    of one dedup group share one CSR)."""
    import ctypes as C
    from paper_2211_05239_b200 import _lib
    lib = _lib.load()
    F, rows, D, B = 3, 3000, 8, 1024
    caps = _lib.i64s([500, 700, 600])
    fake = [C.c_void_p(4096 * (i + 1)) for i in range(8)]
    P = lambda *xs: (C.c_void_p * len(xs))(*[x.value for x in xs])  # noqa: E731
    nb = lib.recd_pool_bwd_scratch_bytes(F, B, D, caps)
    base = 1 << 40
    cs, cr = (C.c_void_p * F)(), (C.c_void_p * F)()
    inv = P(fake[6], fake[6], fake[7])   # features 0 and 1 share an inverse
    rc = lib.recd_pool_bwd_csr(F, B, D, 0, P(fake[0], fake[1], fake[2]), _lib.i64s([rows] * F),
                               P(fake[2], fake[3], fake[4]), P(fake[4], fake[5], fake[0]), caps,
                               fake[6].value, inv, P(fake[7], fake[7], fake[7]), C.c_float(0.1), 1,
                               None, None, None, base, nb, cs, cr)
    assert rc == 0
    for f in range(F):
        assert base <= cs[f] < base + nb and base <= cr[f] < base + nb
    assert cs[0] == cs[1] and cr[0] == cr[1] and cs[2] != cs[0]
    assert cs[2] - cs[0] == 4 * (B + 1) and cr[2] - cr[0] == 4 * B
