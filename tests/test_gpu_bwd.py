"""Backward (segment-reduce + sorted scatter-add + SGD) vs the oracle.

The reference has no backward; the oracle's definition (oracle/embedding.py,
pinned against torch autograd in test_oracle_backward.py) fixes the fp32
order, so the GPU result is compared bit-exactly; the north_star tolerance
(1e-5 relative, atol 1e-5*max|ref|) is asserted as well for clarity."""

import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu

import paper_2211_05239_b200 as R  # noqa: E402


def _session_feature(rng, b, vocab, max_len, dup=0.8):
    vals, offs, pos, state = [], [], 0, None
    for i in range(b):
        if state is None or rng.random() > dup:
            state = rng.integers(0, vocab, size=int(rng.integers(0, max_len + 1)))
        offs.append(pos)
        vals.append(state)
        pos += state.size
    return np.concatenate(vals).astype(np.int64), np.array(offs, np.int64)


def _close(a, b):
    scale = max(float(np.abs(b).max()), 1e-30)
    np.testing.assert_allclose(a, b, rtol=1e-5, atol=1e-5 * scale)


@pytest.mark.parametrize("op", ["sum", "avg"])
@pytest.mark.parametrize("dim", [1, 8, 64, 128])
def test_sparse_grad_matches_oracle(op, dim):
    rng = np.random.default_rng(dim)
    b, rows = 2000, 500
    v, o = _session_feature(rng, b, rows, 12)
    w = rng.uniform(-0.1, 0.1, size=(rows, dim)).astype(np.float32)
    g = rng.standard_normal((b, dim)).astype(np.float32)
    ik = R.kjt_to_ikjt(R.KJT(b, {"k": R.JaggedTensor(v, o)}), ["k"])
    t = R.EmbeddingTable("k", rows, dim, torch.as_tensor(w, device="cuda"))
    [(ids, grads)] = R.pooled_lookup_backward([ik.per_feature["k"]], [t], op,
                                              [torch.as_tensor(g, device="cuda")],
                                              inverses=[ik.inverse_lookup])
    inv, [(uv, uo)] = oracle.build_ikjt_arrays([(v, o)])
    gu = oracle.pool_backward(g, inv, uo.size)
    rid, rg = oracle.sparse_table_grad(gu, uv, uo, op)
    np.testing.assert_array_equal(ids.cpu().numpy(), rid)
    _close(grads.cpu().numpy(), rg)
    np.testing.assert_array_equal(grads.cpu().numpy(), rg)  # same fp32 order -> bit-exact


@pytest.mark.parametrize("op", ["sum", "avg"])
def test_fused_sgd_shared_table_multi_feature(op):
    """cfg1 shape: several keys share ONE table; occurrences are reduced in
    (feature, unique row, position) order."""
    rng = np.random.default_rng(7)
    b, rows, dim, lr = 1500, 300, 64, 0.05
    feats = [_session_feature(rng, b, rows, m) for m in (3, 9, 17)]
    w = rng.uniform(-0.1, 0.1, size=(rows, dim)).astype(np.float32)
    gs = [rng.standard_normal((b, dim)).astype(np.float32) for _ in feats]
    kjt = R.KJT(b, {f"k{i}": R.JaggedTensor(v, o) for i, (v, o) in enumerate(feats)})
    iks = R.kjt_to_ikjts(kjt, [["k0"], ["k1"], ["k2"]])
    wt = torch.as_tensor(w, device="cuda").clone()
    t = R.EmbeddingTable("shared", rows, dim, wt)
    R.pooled_lookup_backward([ik.per_feature[f"k{i}"] for i, ik in enumerate(iks)], [t] * 3, op,
                             [torch.as_tensor(x, device="cuda") for x in gs],
                             inverses=[ik.inverse_lookup for ik in iks], lr=lr)
    # oracle: concatenate the features' occurrences in feature order
    contrib_vals, contrib_rows = [], []
    for (v, o), gg in zip(feats, gs):
        inv, [(uv, uo)] = oracle.build_ikjt_arrays([(v, o)])
        gu = oracle.pool_backward(gg, inv, uo.size)
        lens = np.diff(np.append(uo, uv.size))
        if op == "avg":
            nz = lens > 0
            gu = gu.copy()
            gu[nz] = gu[nz] / lens[nz].astype(np.float32)[:, None]
        contrib_vals.append(uv)
        contrib_rows.append(gu[np.repeat(np.arange(uo.size), lens)])
    allv = np.concatenate(contrib_vals)
    ids, inv_ids = np.unique(allv, return_inverse=True)
    gw = np.zeros((ids.size, dim), np.float32)
    np.add.at(gw, inv_ids, np.concatenate(contrib_rows))
    ref = oracle.sgd_apply(w, ids, gw, lr)
    np.testing.assert_array_equal(wt.cpu().numpy(), ref)


def test_identity_inverse_backward():
    rng = np.random.default_rng(11)
    b, rows, dim = 700, 100, 16
    v, o = _session_feature(rng, b, rows, 5, dup=0.0)
    w = rng.uniform(-0.1, 0.1, size=(rows, dim)).astype(np.float32)
    g = rng.standard_normal((b, dim)).astype(np.float32)
    t = R.EmbeddingTable("k", rows, dim, torch.as_tensor(w, device="cuda"))
    [(ids, grads)] = R.pooled_lookup_backward([R.JaggedTensor(v, o)], [t], "sum",
                                              [torch.as_tensor(g, device="cuda")])
    rid, rg = oracle.sparse_table_grad(g, v, o, "sum")
    np.testing.assert_array_equal(ids.cpu().numpy(), rid)
    np.testing.assert_array_equal(grads.cpu().numpy(), rg)


def test_dedup_and_kjt_backward_agree_within_tolerance():
    """Dedup changes the grad_W summation order (grad_u first), so the two
    paths agree to fp32 tolerance, not bitwise."""
    rng = np.random.default_rng(5)
    b, rows, dim = 3000, 2000, 32
    v, o = _session_feature(rng, b, rows, 20)
    w = torch.as_tensor(rng.uniform(-0.1, 0.1, size=(rows, dim)).astype(np.float32), device="cuda")
    g = torch.as_tensor(rng.standard_normal((b, dim)).astype(np.float32), device="cuda")
    t = R.EmbeddingTable("k", rows, dim, w)
    ik = R.kjt_to_ikjt(R.KJT(b, {"k": R.JaggedTensor(v, o)}), ["k"])
    [(i1, g1)] = R.pooled_lookup_backward([ik.per_feature["k"]], [t], "sum", [g],
                                          inverses=[ik.inverse_lookup])
    [(i2, g2)] = R.pooled_lookup_backward([R.JaggedTensor(v, o)], [t], "sum", [g])
    assert torch.equal(i1, i2)
    _close(g1.cpu().numpy(), g2.cpu().numpy())


def test_module_autograd_fused_sgd():
    rng = np.random.default_rng(2)
    b, rows, dim, lr = 800, 200, 8, 0.1
    v, o = _session_feature(rng, b, rows, 6)
    w0 = rng.uniform(-0.1, 0.1, size=(rows, dim)).astype(np.float32)
    t = R.EmbeddingTable("k", rows, dim, torch.as_tensor(w0, device="cuda").clone())
    ebc = R.DedupEmbeddingBagCollection({"k": t}, "sum", lr=lr)
    ik = R.kjt_to_ikjt(R.KJT(b, {"k": R.JaggedTensor(v, o)}), ["k"])
    out = ebc([ik])["k"]
    ref = oracle.expand(oracle.pooled_lookup(*ik.per_feature["k"].numpy(), w0, "sum"),
                        ik.inverse_lookup.cpu().numpy())
    np.testing.assert_array_equal(out.detach().cpu().numpy(), ref)
    loss = (out * out).sum() * 0.5  # grad_out = out
    loss.backward()
    inv, [(uv, uo)] = oracle.build_ikjt_arrays([(v, o)])
    gu = oracle.pool_backward(ref, inv, uo.size)
    ids, gw = oracle.sparse_table_grad(gu, uv, uo, "sum")
    np.testing.assert_array_equal(t.weights.cpu().numpy(), oracle.sgd_apply(w0, ids, gw, lr))


def test_backward_deterministic():
    rng = np.random.default_rng(8)
    b, rows, dim = 5000, 50, 128
    v, o = _session_feature(rng, b, rows, 30, dup=0.3)
    w = torch.as_tensor(rng.uniform(-0.1, 0.1, size=(rows, dim)).astype(np.float32), device="cuda")
    g = torch.as_tensor(rng.standard_normal((b, dim)).astype(np.float32), device="cuda")
    t = R.EmbeddingTable("k", rows, dim, w)
    ik = R.kjt_to_ikjt(R.KJT(b, {"k": R.JaggedTensor(v, o)}), ["k"])
    res = [R.pooled_lookup_backward([ik.per_feature["k"]], [t], "sum", [g],
                                    inverses=[ik.inverse_lookup])[0][1] for _ in range(3)]
    assert torch.equal(res[0], res[1]) and torch.equal(res[1], res[2])
