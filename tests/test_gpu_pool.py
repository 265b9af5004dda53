"""Pooled lookup + expansion on the GPU vs the reference (golden) / oracle.

The sum follows numpy's reduceat order, so sum/avg/max are compared
bit-exactly (stronger than north_star's 1e-5 relative)."""

import json

import numpy as np
import pytest
import torch

import oracle
from conftest import golden

pytestmark = pytest.mark.gpu

import paper_2211_05239_b200 as R  # noqa: E402


def _table(w, key="t"):
    w = torch.as_tensor(w, device="cuda")
    return R.EmbeddingTable(key, w.shape[0], w.shape[1], w)


@pytest.mark.parametrize("dim", [1, 4, 8, 64, 128])
@pytest.mark.parametrize("op", ["sum", "avg", "max"])
def test_fused_pool_matches_reference_bit_exact(dim, op):
    g = golden("pool")
    t = _table(g[f"d{dim}/weights"])
    jt = R.JaggedTensor(g[f"d{dim}/values"], g[f"d{dim}/offsets"])
    [out] = R.pooled_lookup([jt], [t], op)
    np.testing.assert_array_equal(out.cpu().numpy(), g[f"d{dim}/{op}"])
    inv = torch.as_tensor(g[f"d{dim}/inverse"], device="cuda")
    [exp] = R.pooled_lookup([jt], [t], op, inverses=[inv])
    np.testing.assert_array_equal(exp.cpu().numpy(), g[f"d{dim}/{op}_expanded"])


@pytest.mark.parametrize("dim", [4, 64, 128])
@pytest.mark.parametrize("op", ["sum", "avg", "max"])
def test_dense_pool_and_lookup_match_reference(dim, op):
    g = golden("pool")
    t = _table(g[f"d{dim}/weights"])
    jt = R.JaggedTensor(g[f"d{dim}/values"], g[f"d{dim}/offsets"])
    acts = R.embedding_lookup(jt, t)
    np.testing.assert_array_equal(acts.cpu().numpy(), g[f"d{dim}/weights"][g[f"d{dim}/values"]])
    out = R.pool(acts, jt.offsets, op)
    np.testing.assert_array_equal(out.cpu().numpy(), g[f"d{dim}/{op}"])


def test_errors_match_reference_text():
    msgs = json.loads(str(golden("errors")["json"][0]))
    t = _table(np.arange(4, dtype=np.float32).reshape(-1, 1), "b")
    jt = R.JaggedTensor.from_rows([[1], [9], [3]])
    with pytest.raises(ValueError) as e:
        R.embedding_lookup(jt, t, "b")
    assert str(e.value) == msgs["id_oob"][1]
    with pytest.raises(ValueError) as e:
        R.pooled_lookup([jt], [t], "sum", keys=["b"])
    assert str(e.value) == msgs["id_oob"][1]
    with pytest.raises(ValueError) as e:
        R.pool(torch.zeros((1, 1), device="cuda"), torch.tensor([0]), "median")
    assert str(e.value) == msgs["pool_op"][1]


def test_worked_group_sum():
    """test_trainer_sim.py:94-109: sum pool [24, 21] -> expand [24, 24, 21]."""
    rows = [{"c": [7, 8], "d": [9]}, {"c": [7, 8], "d": [9]}, {"c": [10], "d": [11]}]
    ik = R.build_ikjt(rows, ["c", "d"])
    seq = R.JaggedTensor.from_rows([[7, 8, 9], [10, 11]])
    t = _table(np.arange(12, dtype=np.float32).reshape(-1, 1))
    [out] = R.pooled_lookup([seq], [t], "sum", inverses=[ik.inverse_lookup])
    assert out.cpu().numpy().ravel().tolist() == [24.0, 24.0, 21.0]


@pytest.mark.parametrize("op", ["sum", "avg", "max"])
def test_cfg1_fused_dedup_path_equals_kjt_path(op):
    """The equivalence oracle of the reference (trainer_sim.py:494-496):
    dedup-mode outputs are bit-identical to baseline-mode outputs."""
    from tools.datagen import (SampleCountDist, SessionConfig, cfg1_specs,
                                               generate_clustered_batch)
    batch = generate_clustered_batch(SessionConfig(600, SampleCountDist("geometric", 16.5), 0),
                                     cfg1_specs(), 4096)
    w = torch.empty((1_000_000, 64), device="cuda").uniform_(-0.1, 0.1)
    t = R.EmbeddingTable("shared", 1_000_000, 64, w)
    kjt = R.KJT(4096, {k: R.JaggedTensor(batch.values[k], batch.offsets[k]) for k in batch.keys})
    iks = R.kjt_to_ikjts(kjt, [[k] for k in batch.keys])
    feats = [ik.per_feature[k] for ik, k in zip(iks, batch.keys)]
    ded = R.pooled_lookup(feats, [t] * 8, op, inverses=[ik.inverse_lookup for ik in iks])
    base = R.pooled_lookup([kjt.entries[k] for k in batch.keys], [t] * 8, op)
    wn = w.cpu().numpy()
    for k, d, b in zip(batch.keys, ded, base):
        assert torch.equal(d, b)
        ref = oracle.pooled_lookup(batch.values[k], batch.offsets[k], wn, op)
        np.testing.assert_array_equal(b.cpu().numpy(), ref)


def test_long_rows_pairwise_tree():
    rng = np.random.default_rng(1)
    lens = np.array([0, 1, 2, 7, 8, 9, 128, 129, 130, 255, 256, 257, 1000, 4097], np.int64)
    offs = np.zeros(lens.size, np.int64)
    offs[1:] = np.cumsum(lens[:-1])
    vals = rng.integers(0, 300, size=int(lens.sum())).astype(np.int64)
    w = (rng.standard_normal((300, 128)) * 10.0 ** rng.integers(-3, 3, (300, 1))).astype(np.float32)
    t = _table(w)
    for op in ("sum", "avg", "max"):
        [out] = R.pooled_lookup([R.JaggedTensor(vals, offs)], [t], op)
        np.testing.assert_array_equal(out.cpu().numpy(), oracle.pooled_lookup(vals, offs, w, op))


def _chains(rng, L, nrows, vocab, brk_p):
    """Unique rows of one length L built as chains of one-position shifts
    (row u+1 = row u [1:] + [x]) broken with probability brk_p."""
    rows, cur = [], list(rng.integers(0, vocab, L))
    for _ in range(nrows):
        rows.append(cur)
        if rng.random() < brk_p:
            cur = list(rng.integers(0, vocab, L))
        else:
            cur = cur[1:] + [int(rng.integers(0, vocab))]
    return rows


@pytest.mark.parametrize("L", [2, 3, 8, 9, 128, 129, 256, 300, 512, 513])
@pytest.mark.parametrize("brk_p", [0.0, 0.3, 0.9])
def test_shifted_window_sharing_bit_exact(L, brk_p):
    """Unique rows that are chains of shifted windows (session histories),
    D = 128, sum / avg, long chains, several chains per group of 8 rows,
    chains of one, a partial last group, rows up to 513 long -- bit-exact
    against the oracle's reduceat order."""
    rng = np.random.default_rng(L * 10 + int(brk_p * 10))
    nrows = 8 * 5 + 3
    rows = _chains(rng, L, nrows, 5000, brk_p)
    vals = np.array([v for r in rows for v in r], np.int64)
    offs = np.arange(nrows, dtype=np.int64) * L
    w = (rng.standard_normal((5000, 128)) * 10.0 ** rng.integers(-3, 3, (5000, 1))).astype(np.float32)
    t = _table(w)
    for op in ("sum", "avg"):
        [out] = R.pooled_lookup([R.JaggedTensor(vals, offs)], [t], op)
        np.testing.assert_array_equal(out.cpu().numpy(), oracle.pooled_lookup(vals, offs, w, op))


def test_shifted_window_out_of_range_id():
    """An out-of-range ID as the last ID of a chained (shifted) row raises
    the reference's ValueError."""
    rng = np.random.default_rng(5)
    L = 16
    rows = _chains(rng, L, 16, 100, 0.0)
    vals = np.array([v for r in rows for v in r], np.int64)
    bad = 5 * L + L - 1          # last ID of row 5
    vals[bad] = 100
    offs = np.arange(16, dtype=np.int64) * L
    t = _table(np.ones((100, 128), np.float32))
    with pytest.raises(ValueError) as e:
        R.pooled_lookup([R.JaggedTensor(vals, offs)], [t], "sum")
    assert "100" in str(e.value)
