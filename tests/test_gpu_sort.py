"""The segmented stable radix sort under the backward (recd_sort_pairs)
against numpy's stable argsort: many equal keys (stability), several
segments with device counts below their capacity, 8..32 key bits."""

import ctypes as C

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2211_05239_b200 import _lib  # noqa: E402


@pytest.mark.parametrize("bits,nseg,maxn,dist", [
    (24, 26, 300_000, "dup"), (16, 3, 70_000, "dup"), (8, 1, 5000, "dup"), (32, 4, 40_000, "dup"),
    (24, 64, 9000, "dup"), (20, 2, 1, "dup"),
    # uniform keys over the full digit range, every key in one top digit,
    # 30/32-bit keys (4 passes), many small segments
    (24, 26, 1_200_000, "uniform"), (24, 3, 400_000, "onebucket"), (30, 5, 200_000, "uniform"),
    (32, 2, 300_000, "uniform"), (28, 2, 100_000, "uniform"), (22, 70, 20_000, "uniform")])
def test_sort_pairs_stable(bits, nseg, maxn, dist):
    rng = np.random.default_rng(bits * 100 + nseg)
    caps = rng.integers(1, maxn + 1, size=nseg)
    counts = [int(rng.integers(0, c + 1)) for c in caps]
    bases = np.concatenate([[0], np.cumsum(caps)[:-1]]).astype(np.int64)
    total = int(caps.sum())
    hi = (1 << bits) if bits < 32 else (1 << 32)
    nkeys = max(2, min(hi, 1 + total // 5))          # heavy duplication
    if dist == "uniform":
        nkeys = hi
    keys = rng.integers(0, nkeys, size=total, dtype=np.uint64) % hi
    if dist == "onebucket":  # every key in the same top digit, low bits duplicated
        keys = (np.uint64(5) << np.uint64(bits - 8)) | rng.integers(0, 3000, size=total, dtype=np.uint64)
    if bits < 32:  # bits above `bits` must not affect the order
        keys |= rng.integers(0, 1 << (32 - bits), size=total, dtype=np.uint64) << np.uint64(bits)
    keys = (keys & 0xffffffff).astype(np.uint32)
    vals = np.arange(total, dtype=np.uint32)
    dev = torch.device("cuda")
    k = torch.as_tensor(keys.view(np.int32), device=dev)
    v = torch.as_tensor(vals.view(np.int32), device=dev)
    ka, va = torch.empty_like(k), torch.empty_like(v)
    cnt = [torch.tensor([c], dtype=torch.int64, device=dev) for c in counts]
    lib = _lib.load()
    nb = lib.recd_sort_pairs_scratch_bytes(nseg, _lib.i64s(bases.tolist()), _lib.i64s(caps.tolist()))
    scratch = torch.empty(nb, dtype=torch.uint8, device=dev)
    alt = C.c_int32(-1)
    rc = lib.recd_sort_pairs(nseg, _lib.i64s(bases.tolist()), _lib.i64s(caps.tolist()), _lib.ptrs(cnt),
                             bits, k.data_ptr(), v.data_ptr(), ka.data_ptr(), va.data_ptr(),
                             C.byref(alt), scratch.data_ptr(), nb, _lib.stream_ptr(dev))
    assert rc == 0
    torch.cuda.synchronize()
    rk, rv = (ka, va) if alt.value else (k, v)
    rk = rk.cpu().numpy().view(np.uint32)
    rv = rv.cpu().numpy().view(np.uint32)
    mask = np.uint32((1 << bits) - 1) if bits < 32 else np.uint32(0xffffffff)
    for s in range(nseg):
        a, n = int(bases[s]), counts[s]
        seg_k = keys[a:a + n]
        order = np.argsort(seg_k & mask, kind="stable")
        np.testing.assert_array_equal(rv[a:a + n], vals[a:a + n][order])
        np.testing.assert_array_equal(rk[a:a + n], seg_k[order])


def _sort_and_check(keys, caps, counts, bits):
    dev = torch.device("cuda")
    nseg = len(caps)
    caps = np.asarray(caps, np.int64)
    bases = np.concatenate([[0], np.cumsum(caps)[:-1]]).astype(np.int64)
    vals = np.arange(keys.size, dtype=np.uint32)
    k = torch.as_tensor(keys.view(np.int32), device=dev)
    v = torch.as_tensor(vals.view(np.int32), device=dev)
    ka, va = torch.empty_like(k), torch.empty_like(v)
    cnt = [torch.tensor([c], dtype=torch.int64, device=dev) for c in counts]
    lib = _lib.load()
    nb = lib.recd_sort_pairs_scratch_bytes(nseg, _lib.i64s(bases.tolist()), _lib.i64s(caps.tolist()))
    scratch = torch.empty(nb, dtype=torch.uint8, device=dev)
    alt = C.c_int32(-1)
    rc = lib.recd_sort_pairs(nseg, _lib.i64s(bases.tolist()), _lib.i64s(caps.tolist()), _lib.ptrs(cnt),
                             bits, k.data_ptr(), v.data_ptr(), ka.data_ptr(), va.data_ptr(),
                             C.byref(alt), scratch.data_ptr(), nb, _lib.stream_ptr(dev))
    assert rc == 0
    torch.cuda.synchronize()
    rk, rv = (ka, va) if alt.value else (k, v)
    rk = rk.cpu().numpy().view(np.uint32)
    rv = rv.cpu().numpy().view(np.uint32)
    for s in range(nseg):
        a, n = int(bases[s]), counts[s]
        order = np.argsort(keys[a:a + n] & np.uint32((1 << bits) - 1), kind="stable")
        np.testing.assert_array_equal(rv[a:a + n], vals[a:a + n][order])


def test_sort_interleaved_tickets_skewed_segments():
    """Tickets interleaved over the segments in proportion to their tile
    counts (>= 64 tiles per segment on average): segments of very different
    sizes, empty ones, a one-element one, partial last tiles, clustered
    (history-like) and random keys -- every segment stable-sorted."""
    rng = np.random.default_rng(11)
    caps = [2_000_000, 1, 0, 4097, 700_000, 1_500_000, 3, 260_000]
    counts = [2_000_000, 1, 0, 4097, 699_999, 1_234_567, 0, 260_000]
    caps = [max(c, 1) for c in caps]
    keys = rng.integers(0, 10_000_000, size=sum(caps), dtype=np.uint64).astype(np.uint32)
    keys[: 2_000_000] = np.repeat(rng.integers(0, 10_000_000, 2_000_000 // 8), 8)  # clustered equal keys
    _sort_and_check(keys, caps, counts, 24)
