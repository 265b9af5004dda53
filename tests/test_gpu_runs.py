"""The backward's diagonal-run occurrences (csrc/recd_bwd.cu k_rv*): one
sort element per run of an ID through shifted history windows.  Bit-exact
against the oracle's (unique row, position)-ordered scatter-add on the
cases that stress the exactness argument: IDs repeated inside a row (dirty
rows, overlapping diagonals), a padding ID in every row, rows longer than the
duplicate-check limit, shared tables, and runs that end at row/batch edges."""

import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu

import paper_2211_05239_b200 as R  # noqa: E402


@pytest.fixture(autouse=True, params=["runs", "values"])
def occurrences(request, monkeypatch):
    """Both occurrence encodings of the backward: diagonal runs
    (RECD_BWD_RUNS=1, read by librecd per call) and one element per value."""
    monkeypatch.setenv("RECD_BWD_RUNS", "1" if request.param == "runs" else "0")
    return request.param


def _windows(rng, b, vocab, length, p_shift=0.3, pad=0, pad_id=0, var_len=False):
    """Session-like rows: each row is the previous one shifted by one (new ID
    at the end) with probability p_shift, else identical or a new session."""
    rows, hist = [], list(rng.integers(0, vocab, size=length))
    for i in range(b):
        x = rng.random()
        if x < p_shift:
            hist = hist[1:] + [int(rng.integers(0, vocab))]
        elif x > 0.97:
            hist = list(rng.integers(0, vocab, size=length))
        row = [int(v) for v in hist]
        if var_len and rng.random() < 0.2:
            row = row[: int(rng.integers(0, length + 1))]
        if pad:
            row = row[: max(0, len(row) - pad)] + [pad_id] * pad
        rows.append(row)
    offs = np.cumsum([0] + [len(r) for r in rows[:-1]]).astype(np.int64)
    vals = np.array([v for r in rows for v in r], dtype=np.int64)
    return vals, offs


def _check(feats, rows, dim, op="sum", seed=0):
    """feats: [(values, offsets)] sharing one table; sparse grads vs oracle."""
    rng = np.random.default_rng(seed)
    b = feats[0][1].size
    w = rng.uniform(-0.1, 0.1, size=(rows, dim)).astype(np.float32)
    t = R.EmbeddingTable("t", rows, dim, torch.as_tensor(w, device="cuda"))
    jts, invs, grads, contrib_v, contrib_g = [], [], [], [], []
    for f, (v, o) in enumerate(feats):
        ik = R.kjt_to_ikjt(R.KJT(b, {f"k{f}": R.JaggedTensor(v, o)}), [f"k{f}"])
        g = rng.standard_normal((b, dim)).astype(np.float32)
        jts.append(ik.per_feature[f"k{f}"])
        invs.append(ik.inverse_lookup)
        grads.append(torch.as_tensor(g, device="cuda"))
        inv, [(uv, uo)] = oracle.build_ikjt_arrays([(v, o)])
        gu = oracle.pool_backward(g, inv, uo.size)
        lens = np.diff(np.append(uo, uv.size))
        rowid = np.repeat(np.arange(uo.size), lens)
        contrib_v.append(uv)
        contrib_g.append(gu[rowid] if op == "sum" else
                         (gu / np.maximum(lens, 1).astype(np.float32)[:, None])[rowid])
    [(ids, gw)] = R.pooled_lookup_backward(jts, [t] * len(feats), op, grads, inverses=invs)
    allv = np.concatenate(contrib_v)
    rid, inv_ids = np.unique(allv, return_inverse=True)
    rg = np.zeros((rid.size, dim), np.float32)
    np.add.at(rg, inv_ids, np.concatenate(contrib_g))   # (feature, row, position) order
    np.testing.assert_array_equal(ids.cpu().numpy(), rid)
    np.testing.assert_array_equal(gw.cpu().numpy(), rg)


@pytest.mark.parametrize("vocab", [7, 40, 100000])
@pytest.mark.parametrize("length", [3, 16, 64])
def test_shifted_windows(vocab, length):
    rng = np.random.default_rng(vocab * 1000 + length)
    _check([_windows(rng, 3000, vocab, length)], max(vocab, 8), 32, seed=length)


@pytest.mark.parametrize("pad", [1, 4])
def test_padding_id_in_every_row(pad):
    rng = np.random.default_rng(pad)
    _check([_windows(rng, 4000, 5000, 24, pad=pad, var_len=True)], 5000, 16, seed=pad)


def test_rows_longer_than_duplicate_check():
    rng = np.random.default_rng(3)
    _check([_windows(rng, 400, 300, 700)], 300, 8)


@pytest.mark.parametrize("op", ["sum", "avg"])
def test_shared_table_features(op):
    rng = np.random.default_rng(9)
    feats = [_windows(rng, 2000, 60, L, var_len=True) for L in (5, 12, 33)]
    _check(feats, 60, 16, op=op, seed=2)


def test_step_fused_sgd():
    """Step-level: the fused SGD through TrainStep equals the oracle with either
    occurrence encoding."""
    from paper_2211_05239_b200.step import TrainStep
    rng = np.random.default_rng(4)
    b, rows, dim, lr = 2048, 300, 32, 0.1
    keys = ["a", "b"]
    data = {k: _windows(rng, b, rows, L) for k, L in zip(keys, (8, 48))}
    w0 = {k: rng.uniform(-0.1, 0.1, size=(rows, dim)).astype(np.float32) for k in keys}
    tables = {k: R.EmbeddingTable(k, rows, dim, torch.as_tensor(w0[k], device="cuda").clone())
              for k in keys}
    step = TrainStep([[k] for k in keys], b, {k: data[k][0].size for k in keys}, tables, "sum", lr)
    step.load_batch({k: data[k][0] for k in keys}, {k: data[k][1] for k in keys})
    step.fill_grad_out(5)
    step.run()
    torch.cuda.synchronize()
    for f, k in enumerate(keys):
        v, o = data[k]
        inv, [(uv, uo)] = oracle.build_ikjt_arrays([(v, o)])
        gu = oracle.pool_backward(step.grad_out[f].cpu().numpy(), inv, uo.size)
        ids, g = oracle.sparse_table_grad(gu, uv, uo, "sum")
        want = w0[k].copy()
        want[ids] = w0[k][ids] - (np.float32(lr) * g).astype(np.float32)
        np.testing.assert_array_equal(tables[k].weights.cpu().numpy(), want)
