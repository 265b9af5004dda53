"""Device decode of row-delta coded KJT rows (recd_rowcode_decode) against
the host values: session batches with fixed- and variable-length keys, the
edge rows of tests/test_rowcode.py, and the H2D pipeline end to end."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2211_05239_b200 import _lib, rowcode  # noqa: E402
from tools.datagen import (FeatureSpec, SampleCountDist, SessionConfig,  # noqa: E402
                           generate_clustered_batch)


def _decode(vals, offs, caps=None):
    F, B = len(vals), offs[0].size
    codes = [np.empty(B, np.uint8) for _ in vals]
    lits = [np.empty(max(v.size, 1), np.int64) for v in vals]
    cnt = rowcode.encode(vals, offs, B, codes, lits)
    dev = torch.device("cuda")
    caps = caps or [max(v.size, 1) for v in vals]
    d_codes = [torch.as_tensor(c, device=dev) for c in codes]
    d_offs = [torch.as_tensor(o, device=dev) for o in offs]
    d_lits = [torch.as_tensor(l[: max(n, 1)], device=dev) for l, n in zip(lits, cnt)]
    d_nv = torch.tensor([v.size for v in vals], dtype=torch.int64, device=dev)
    out = [torch.full((c,), -7, dtype=torch.int64, device=dev) for c in caps]
    lib = _lib.load()
    nb = lib.recd_rowcode_scratch_bytes(F, B)
    scratch = torch.empty(nb, dtype=torch.uint8, device=dev)
    rc = lib.recd_rowcode_decode(F, B, _lib.ptrs(d_codes), _lib.ptrs(d_offs), d_nv.data_ptr(),
                                 _lib.i64s(caps), _lib.ptrs(d_lits), _lib.ptrs(out),
                                 scratch.data_ptr(), nb, _lib.stream_ptr(dev))
    assert rc == 0
    torch.cuda.synchronize()
    for f, v in enumerate(vals):
        got = out[f].cpu().numpy()
        np.testing.assert_array_equal(got[: v.size], v)
        assert (got[v.size:] == -7).all()


@pytest.mark.parametrize("b", [1, 1000, 65536])
def test_decode_session_batch(b):
    specs = [FeatureSpec(f"k{i}", "user_sequence", float(L), 10_000_000, 0.15)
             for i, L in enumerate([1, 8, 40, 256])]
    specs.append(FeatureSpec("item", "item", 7.3, 1000))
    bt = generate_clustered_batch(SessionConfig(max(2, b // 8), SampleCountDist("geometric", 16.5), 5),
                                  specs, b)
    vals = [bt.values[k] for k in bt.keys]
    offs = [bt.offsets[k] for k in bt.keys]
    _decode(vals, offs, caps=[v.size + 17 for v in vals])


def test_decode_edge_rows():
    rows = [[], [], [5], [5], [6], [1, 2, 3], [2, 3, 4], [2, 3, 4], [3, 4], [3, 4, 9], [4, 9, 9],
            [9, 9, 9], [9, 9, 9], [], [7], [7, 7], [7, 7]]
    offs = np.cumsum([0] + [len(r) for r in rows[:-1]]).astype(np.int64)
    vals = np.array([x for r in rows for x in r], dtype=np.int64)
    _decode([vals, vals[::-1].copy()], [offs, offs])


def test_random_rows_tiny_vocab():
    rng = np.random.default_rng(1)
    B = 5000
    vals, offs = [], []
    for f in range(3):
        lens = rng.integers(0, 9, size=B)
        vals.append(rng.integers(0, 2, size=int(lens.sum())).astype(np.int64))
        offs.append(np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.int64))
    _decode(vals, offs)
