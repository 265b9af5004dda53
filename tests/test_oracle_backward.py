"""The backward oracle (our definition; the reference has none) agrees with
torch-CPU autograd of F.embedding_bag over the expanded KJT."""

import numpy as np
import pytest
import torch

import oracle


def _case(seed, b=300, rows=200, dim=16, vocab=40):
    rng = np.random.default_rng(seed)
    feats, state = [], None
    vals, offs = [], []
    pos = 0
    for i in range(b):
        if state is None or rng.random() > 0.7:
            state = rng.integers(0, vocab, size=int(rng.integers(0, 9)))
        offs.append(pos)
        vals.append(state)
        pos += state.size
    v = np.concatenate(vals).astype(np.int64)
    o = np.array(offs, dtype=np.int64)
    w = rng.uniform(-0.1, 0.1, size=(rows, dim)).astype(np.float32)
    g = rng.standard_normal((b, dim)).astype(np.float32)
    return v, o, w, g


@pytest.mark.parametrize("op", ["sum", "avg"])
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_backward_oracle_vs_torch_autograd(op, seed):
    v, o, w, g = _case(seed)
    inv, [(uv, uo)] = oracle.build_ikjt_arrays([(v, o)])
    u = uo.size
    gu = oracle.pool_backward(g, inv, u)
    ids, gw = oracle.sparse_table_grad(gu, uv, uo, op)

    wt = torch.tensor(w, dtype=torch.float64, requires_grad=True)
    out = torch.nn.functional.embedding_bag(
        torch.tensor(v), wt, torch.tensor(o), mode="sum" if op == "sum" else "mean",
        include_last_offset=False)
    out.backward(torch.tensor(g, dtype=torch.float64))
    dense = wt.grad.numpy()
    ref = dense[ids]
    scale = np.abs(ref).max()
    np.testing.assert_allclose(gw, ref, rtol=1e-5, atol=1e-5 * scale)
    # rows never touched get no gradient
    untouched = np.setdiff1d(np.arange(w.shape[0]), ids)
    assert np.all(dense[untouched] == 0)


def test_forward_oracle_vs_torch_embedding_bag():
    v, o, w, _ = _case(5)
    inv, [(uv, uo)] = oracle.build_ikjt_arrays([(v, o)])
    for op, mode in (("sum", "sum"), ("avg", "mean"), ("max", "max")):
        out = oracle.expand(oracle.pooled_lookup(uv, uo, w, op), inv)
        ref = torch.nn.functional.embedding_bag(torch.tensor(v), torch.tensor(w),
                                                torch.tensor(o), mode=mode).numpy()
        np.testing.assert_allclose(out, ref, rtol=1e-5, atol=1e-5 * np.abs(ref).max())


def test_sgd_apply_separately_rounded():
    w = np.array([[1.0, 2.0], [3.0, 4.0]], dtype=np.float32)
    out = oracle.sgd_apply(w, np.array([1]), np.array([[0.5, -1.0]], dtype=np.float32), 0.1)
    np.testing.assert_array_equal(out[0], w[0])
    np.testing.assert_array_equal(out[1], w[1] - np.float32(0.1) * np.array([0.5, -1.0], np.float32))
