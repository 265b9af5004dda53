"""TrainStep (the bench's step: dedup -> pooled lookup -> expand -> backward
with fused SGD) against the oracle, eagerly and as a CUDA graph, with the
backward's prepare half overlapped on a side stream and without.  Session
batches from the restated reference generator give consecutive unique rows
that share IDs (shifted history windows), which is what the scatter's
sequential-prefix rows exploit; results must stay bit-exact."""

import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu

import paper_2211_05239_b200 as R  # noqa: E402
from tools.datagen import (FeatureSpec, SampleCountDist, SessionConfig,  # noqa: E402
                                           generate_clustered_batch)
from paper_2211_05239_b200.step import TrainStep  # noqa: E402


def _batch(b, lens, vocab, seed, mean=16.5, change=0.15):
    specs = [FeatureSpec(f"k{i}", "user_sequence", float(L), vocab, change) for i, L in enumerate(lens)]
    return generate_clustered_batch(SessionConfig(max(1, b // 8), SampleCountDist("geometric", mean), seed),
                                    specs, b)


def _oracle_step(batch, w0s, grads, lr):
    """Per key: dedup, pooled sum + expand, backward, SGD on that key's table."""
    outs, w1s = {}, {}
    for k in batch.keys:
        v, o = batch.values[k], batch.offsets[k]
        inv, [(uv, uo)] = oracle.build_ikjt_arrays([(v, o)])
        outs[k] = oracle.expand(oracle.pooled_lookup(uv, uo, w0s[k], "sum"), inv)
        gu = oracle.pool_backward(grads[k], inv, uo.size)
        ids, g = oracle.sparse_table_grad(gu, uv, uo, "sum")
        w1 = w0s[k].copy()
        w1[ids] = w0s[k][ids] - (np.float32(lr) * g).astype(np.float32)
        w1s[k] = w1
    return outs, w1s


@pytest.mark.parametrize("fused", ["0", "1"])
@pytest.mark.parametrize("overlap", [True, False])
@pytest.mark.parametrize("graph", [True, False])
def test_train_step_matches_oracle(overlap, graph, fused, monkeypatch):
    """fused: the lookup expands through the backward's inverse CSR
    (recd_pool_fwd_csr) instead of k_expand."""
    monkeypatch.setenv("RECD_FUSED_EXPAND", fused)
    b, vocab, dim, lr = 2048, 5000, 128, 0.05
    batch = _batch(b, [4, 24, 64], vocab, seed=3)
    keys = list(batch.keys)
    rng = np.random.default_rng(0)
    w0s = {k: rng.uniform(-0.1, 0.1, size=(vocab, dim)).astype(np.float32) for k in keys}
    tables = {k: R.EmbeddingTable(k, vocab, dim, torch.as_tensor(w0s[k], device="cuda").clone())
              for k in keys}
    caps = {k: int(batch.values[k].size) for k in keys}
    step = TrainStep([[k] for k in keys], b, caps, tables, "sum", lr, "dedup", overlap=overlap)
    step.load_batch(batch.values, batch.offsets)
    grads = {k: rng.standard_normal((b, dim)).astype(np.float32) for k in keys}
    for f, k in enumerate(keys):
        step.grad_out[f].copy_(torch.as_tensor(grads[k]))
    if graph:
        # capture runs the step once (warm-up) before recording: restore the tables after
        step.capture()
        for k in keys:
            tables[k].weights.copy_(torch.as_tensor(w0s[k]))
        step.replay()
    else:
        step.run()
    torch.cuda.synchronize()
    outs, w1s = _oracle_step(batch, w0s, grads, lr)
    for f, k in enumerate(keys):
        np.testing.assert_array_equal(step.out[f].cpu().numpy(), outs[k])
        np.testing.assert_array_equal(tables[k].weights.cpu().numpy(), w1s[k])


def test_long_sessions_many_consecutive_rows():
    """Fixed 64-sample sessions with frequent window shifts: runs of consecutive
    unique rows far longer than the prefix rows cover."""
    b, vocab, dim, lr = 4096, 20000, 64, 0.1
    batch = _batch(b, [32, 128], vocab, seed=11, mean=64, change=0.6)
    keys = list(batch.keys)
    rng = np.random.default_rng(1)
    w0s = {k: rng.uniform(-0.1, 0.1, size=(vocab, dim)).astype(np.float32) for k in keys}
    tables = {k: R.EmbeddingTable(k, vocab, dim, torch.as_tensor(w0s[k], device="cuda").clone())
              for k in keys}
    caps = {k: int(batch.values[k].size) for k in keys}
    step = TrainStep([[k] for k in keys], b, caps, tables, "sum", lr, "dedup")
    step.load_batch(batch.values, batch.offsets)
    grads = {k: rng.standard_normal((b, dim)).astype(np.float32) for k in keys}
    for f, k in enumerate(keys):
        step.grad_out[f].copy_(torch.as_tensor(grads[k]))
    step.run()
    torch.cuda.synchronize()
    _, w1s = _oracle_step(batch, w0s, grads, lr)
    for k in keys:
        np.testing.assert_array_equal(tables[k].weights.cpu().numpy(), w1s[k])


@pytest.mark.parametrize("bad", ["rows", "negative", "huge"])
@pytest.mark.parametrize("graph", [False, True])
def test_out_of_range_id_reports_and_leaves_tables_intact(bad, graph):
    """An ID outside [0, rows) (e.g. the reader's clamp transform with
    param=rows) is the reference's ValueError (trainer_sim.py:312-320); the
    fused SGD must not touch any table row for that batch (k_occ flags the ID,
    k_scatter skips), and TrainStep.check() raises the reference's text."""
    b, vocab, dim, lr = 512, 3000, 64, 0.5
    batch = _batch(b, [8, 16], vocab, seed=5)
    keys = list(batch.keys)
    bad_id = {"rows": vocab, "negative": -3, "huge": (1 << 40) + 7}[bad]
    vals = {k: batch.values[k].copy() for k in keys}
    vals[keys[1]][37] = bad_id
    rng = np.random.default_rng(2)
    w0s = {k: rng.uniform(-0.1, 0.1, size=(vocab, dim)).astype(np.float32) for k in keys}
    tables = {k: R.EmbeddingTable(k, vocab, dim, torch.as_tensor(w0s[k], device="cuda").clone())
              for k in keys}
    caps = {k: int(batch.values[k].size) for k in keys}
    step = TrainStep([[k] for k in keys], b, caps, tables, "sum", lr, "dedup")
    step.load_batch(vals, batch.offsets)
    step.fill_grad_out(3)
    if graph:
        step.capture()
        step.replay()
    else:
        step.run()
    torch.cuda.synchronize()
    with pytest.raises(ValueError, match=rf"feature '{keys[1]}': ID {bad_id} at position \d+ "
                                         rf"out of range \[0, {vocab}\)"):
        step.check()
    for k in keys[1:]:
        np.testing.assert_array_equal(tables[k].weights.cpu().numpy(), w0s[k])
    # a clean batch afterwards trains normally (the flag is per step)
    step.load_batch(batch.values, batch.offsets)
    step.run()
    torch.cuda.synchronize()
    step.check()
    assert not np.array_equal(tables[keys[1]].weights.cpu().numpy(), w0s[keys[1]])


def test_module_deferred_checks():
    """DedupEmbeddingBagCollection(defer_checks=True): forward + backward never
    read the device; check() raises the reference's error afterwards and the
    fused SGD left the table untouched for that batch."""
    b, vocab, dim = 256, 1000, 16
    batch = _batch(b, [6], vocab, seed=9)
    k = batch.keys[0]
    vals = batch.values[k].copy()
    vals[11] = vocab + 5
    w0 = np.random.default_rng(0).uniform(-0.1, 0.1, size=(vocab, dim)).astype(np.float32)
    t = R.EmbeddingTable(k, vocab, dim, torch.as_tensor(w0, device="cuda").clone())
    ebc = R.DedupEmbeddingBagCollection({k: t}, "sum", lr=0.1, defer_checks=True)
    ik = R.kjt_to_ikjt(R.KJT(b, {k: R.JaggedTensor(vals, batch.offsets[k])}), [k])
    out = ebc(ik)
    out[k].sum().backward()
    torch.cuda.synchronize()
    with pytest.raises(ValueError, match=rf"feature '{k}': ID {vocab + 5} at position \d+ "
                                         rf"out of range \[0, {vocab}\)"):
        ebc.check()
    np.testing.assert_array_equal(t.weights.cpu().numpy(), w0)
    ebc.check()   # errors are reported once


def test_pool_fwd_csr_writes_batch_rows_and_pooled():
    """recd_pool_fwd_csr with a pooled buffer as well: both outputs equal the
    oracle's pooled rows and their expansion."""
    import ctypes as C

    from paper_2211_05239_b200 import _lib
    b, vocab, dim = 1024, 3000, 64
    batch = _batch(b, [6, 40], vocab, seed=11)
    keys = list(batch.keys)
    rng = np.random.default_rng(5)
    w0s = {k: rng.uniform(-0.1, 0.1, size=(vocab, dim)).astype(np.float32) for k in keys}
    tables = {k: R.EmbeddingTable(k, vocab, dim, torch.as_tensor(w0s[k], device="cuda").clone())
              for k in keys}
    caps = {k: int(batch.values[k].size) for k in keys}
    step = TrainStep([[k] for k in keys], b, caps, tables, "sum", 0.0, "dedup")
    step.load_batch(batch.values, batch.offsets)
    s = torch.cuda.current_stream().cuda_stream
    step.dedup(s)
    step.backward_stages(_lib.BWD_INVERSE, s)
    a = step.args()
    cs, cr = step._csr()
    pooled = [torch.full((b, dim), float("nan"), device="cuda") for _ in keys]
    out = [torch.full((b, dim), float("nan"), device="cuda") for _ in keys]
    rc = step.lib.recd_pool_fwd_csr(step.F, b, dim, 0, a.tables, a.rows, a.feat_vals, a.feat_offs,
                                    a.counts_ptr, cs, cr, _lib.ptrs(pooled), _lib.ptrs(out),
                                    step._st(None).err.data_ptr(), s)
    assert rc == 0
    torch.cuda.synchronize()
    for f, k in enumerate(keys):
        inv, [(uv, uo)] = oracle.build_ikjt_arrays([(batch.values[k], batch.offsets[k])])
        ref = oracle.pooled_lookup(uv, uo, w0s[k], "sum")
        np.testing.assert_array_equal(pooled[f][: uo.size].cpu().numpy(), ref)
        np.testing.assert_array_equal(out[f].cpu().numpy(), oracle.expand(ref, inv))
    assert C.c_void_p(cs[0]).value is not None


@pytest.mark.parametrize("fused", ["0", "1"])
@pytest.mark.parametrize("graph", [True, False])
def test_mixed_dedup_and_plain_keys(graph, fused, monkeypatch):
    """One step over deduplicated groups and plain KJT keys together
    (trainer_sim.py:562-574): the dedup'd keys match the oracle's IKJT path,
    the plain key the oracle with an identity inverse (one unique row per
    batch row, gradients reduced per batch row), tables and outputs
    bit-exact, eager and as one CUDA graph."""
    monkeypatch.setenv("RECD_FUSED_EXPAND", fused)
    b, vocab, dim, lr = 2048, 5000, 128, 0.05
    batch = _batch(b, [8, 24, 16], vocab, seed=5)
    keys = list(batch.keys)
    plain = [keys[2]]
    rng = np.random.default_rng(1)
    w0s = {k: rng.uniform(-0.1, 0.1, size=(vocab, dim)).astype(np.float32) for k in keys}
    tables = {k: R.EmbeddingTable(k, vocab, dim, torch.as_tensor(w0s[k], device="cuda").clone())
              for k in keys}
    caps = {k: int(batch.values[k].size) for k in keys}
    step = TrainStep([[keys[0]], [keys[1]]], b, caps, tables, "sum", lr, "dedup", plain=plain)
    assert step.keys == keys
    step.load_batch(batch.values, batch.offsets)
    grads = {k: rng.standard_normal((b, dim)).astype(np.float32) for k in keys}
    for f, k in enumerate(step.keys):
        step.grad_out[f].copy_(torch.as_tensor(grads[k]))
    if graph:
        step.capture()
        for k in keys:
            tables[k].weights.copy_(torch.as_tensor(w0s[k]))
        step.replay()
    else:
        step.run()
    torch.cuda.synchronize()
    outs, w1s = _oracle_step(batch, w0s, grads, lr)
    for k in plain:  # identity inverse: no dedup
        v, o = batch.values[k], batch.offsets[k]
        outs[k] = oracle.pooled_lookup(v, o, w0s[k], "sum")
        ids, g = oracle.sparse_table_grad(grads[k], v, o, "sum")
        w1 = w0s[k].copy()
        w1[ids] = w0s[k][ids] - (np.float32(lr) * g).astype(np.float32)
        w1s[k] = w1
    for f, k in enumerate(step.keys):
        np.testing.assert_array_equal(step.out[f].cpu().numpy(), outs[k])
        np.testing.assert_array_equal(tables[k].weights.cpu().numpy(), w1s[k])
    c = step.host_counts()
    assert c.U[2] == b and c.N_u[2] == batch.values[keys[2]].size
    with pytest.raises(ValueError):
        TrainStep([[keys[0]]], b, caps, tables, "sum", lr, "dedup", plain=[keys[0]])
