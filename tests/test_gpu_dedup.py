"""KJT -> IKJT on the GPU vs the reference (golden) and the oracle: bit-exact."""

import numpy as np
import pytest
import torch

import oracle
from conftest import dedup_cases, golden

pytestmark = pytest.mark.gpu

import paper_2211_05239_b200 as R  # noqa: E402
from paper_2211_05239_b200 import _lib  # noqa: E402


def _kjt(feats, names=None):
    names = names or [f"f{i}" for i in range(len(feats))]
    b = len(feats[0][1])
    return R.KJT(b, {n: R.JaggedTensor(v, o) for n, (v, o) in zip(names, feats)}), names


def _check(ik, names, inv_ref, outs_ref):
    np.testing.assert_array_equal(ik.inverse_lookup.cpu().numpy(), inv_ref)
    for n, (rv, ro) in zip(names, outs_ref):
        v, o = ik.per_feature[n].numpy()
        np.testing.assert_array_equal(v, rv)
        np.testing.assert_array_equal(o, ro)


CASES = list(dedup_cases())


@pytest.mark.parametrize("case", CASES, ids=lambda c: c[0])
def test_dedup_matches_reference_golden(case):
    name, feats, inv_ref, outs_ref = case
    kjt, names = _kjt(feats)
    ik = R.kjt_to_ikjt(kjt, names)
    _check(ik, names, inv_ref, outs_ref)


@pytest.mark.parametrize("mask", [0x1, 0x3, 0xFF])
def test_forced_hash_collisions_stay_exact(mask):
    """Weakened hash: almost every head collides; the exact fallback must
    still reproduce the reference (full compare, tensors.py:270-276)."""
    _lib.set_hash_mask(mask)
    try:
        for name, feats, inv_ref, outs_ref in CASES[:30]:
            kjt, names = _kjt(feats)
            _check(R.kjt_to_ikjt(kjt, names), names, inv_ref, outs_ref)
    finally:
        _lib.set_hash_mask(~0)


def test_batched_groups_one_call_equals_per_group():
    rng = np.random.default_rng(3)
    b = 3000
    feats = []
    for k in range(7):
        vals, offs, pos, state = [], [], 0, None
        for i in range(b):
            if state is None or rng.random() > 0.8:
                state = rng.integers(0, 5 + 3 * k, size=int(rng.integers(0, 6)))
            offs.append(pos)
            vals.append(state)
            pos += state.size
        feats.append((np.concatenate(vals).astype(np.int64), np.array(offs, np.int64)))
    kjt, names = _kjt(feats)
    groups = [names[0:1], names[1:3], names[3:4], names[4:7]]
    iks = R.kjt_to_ikjts(kjt, groups)
    for g, ik in zip(groups, iks):
        gi = [names.index(n) for n in g]
        inv, outs = oracle.build_ikjt_arrays([feats[i] for i in gi])
        _check(ik, g, inv, outs)


def test_cfg1_all_keys_bit_exact():
    from tools.datagen import (SampleCountDist, SessionConfig, cfg1_specs,
                                               generate_clustered_batch)
    g = golden("datagen")
    batch = generate_clustered_batch(SessionConfig(600, SampleCountDist("geometric", 16.5), 0),
                                     cfg1_specs(), 4096)
    kjt = R.KJT(4096, {k: R.JaggedTensor(batch.values[k], batch.offsets[k]) for k in batch.keys})
    iks = R.kjt_to_ikjts(kjt, [[k] for k in batch.keys])
    for k, ik in zip(batch.keys, iks):
        np.testing.assert_array_equal(ik.inverse_lookup.cpu().numpy(), g[f"cfg1/{k}/inverse"])
        v, o = ik.per_feature[k].numpy()
        np.testing.assert_array_equal(v, g[f"cfg1/{k}/uvalues"])
        np.testing.assert_array_equal(o, g[f"cfg1/{k}/uoffsets"])


@pytest.mark.parametrize("b", [1, 2, 255, 256, 257, 16383, 16384, 16385, 65536])
def test_sizes_and_tiles_vs_oracle(b):
    rng = np.random.default_rng(b)
    vals, offs, pos, state = [], [], 0, None
    for i in range(b):
        if state is None or rng.random() > 0.7:
            state = rng.integers(0, 30, size=int(rng.integers(0, 4)))
        offs.append(pos)
        vals.append(state)
        pos += state.size
    v = np.concatenate(vals).astype(np.int64) if vals else np.empty(0, np.int64)
    o = np.array(offs, np.int64)
    kjt, names = _kjt([(v, o)])
    ik = R.kjt_to_ikjt(kjt, names)
    inv, outs = oracle.build_ikjt_arrays([(v, o)])
    _check(ik, names, inv, outs)


def test_long_rows_and_empty_rows():
    rng = np.random.default_rng(9)
    rows = []
    for i in range(500):
        r = rng.random()
        if r < 0.2:
            rows.append(np.empty(0, np.int64))
        elif r < 0.4 and rows:
            rows.append(rows[-1])
        elif r < 0.5 and len(rows) > 10:
            rows.append(rows[int(rng.integers(0, len(rows)))])
        else:
            rows.append(rng.integers(0, 7, size=int(rng.integers(1, 700))))
    lens = np.array([r.size for r in rows])
    o = np.zeros(len(rows), np.int64)
    o[1:] = np.cumsum(lens[:-1])
    v = np.concatenate(rows).astype(np.int64)
    kjt, names = _kjt([(v, o), (v[::-1].copy(), o)])
    ik = R.kjt_to_ikjt(kjt, names[:1])
    inv, outs = oracle.build_ikjt_arrays([(v, o)])
    _check(ik, names[:1], inv, outs)


def test_deterministic_across_runs():
    name, feats, inv_ref, outs_ref = CASES[-1]
    kjt, names = _kjt(feats)
    a = R.kjt_to_ikjt(kjt, names)
    for _ in range(3):
        b = R.kjt_to_ikjt(kjt, names)
        assert torch.equal(a.inverse_lookup, b.inverse_lookup)


def test_build_ikjt_from_rows_and_errors():
    rows = [{"a": [1, 2], "b": [3, 4, 5]}, {"a": [], "b": [4, 5, 6]}, {"a": [1, 2], "b": [3, 4, 5]}]
    ik = R.build_ikjt(rows, ["b"])
    assert ik.inverse_lookup.cpu().tolist() == [0, 1, 0]
    assert ik.per_feature["b"].to_pylists() == [[3, 4, 5], [4, 5, 6]]
    with pytest.raises(ValueError, match="empty batch"):
        R.build_ikjt([], ["a"])
    with pytest.raises(ValueError, match="empty dedup group"):
        R.build_ikjt(rows, [])
