"""cfg2 at full size (B = 65,536, 26 keys, lists up to 256 IDs, 133.7 M KJT
values) through size-independent properties (the oracle is too slow for the
whole batch): the IKJT expands back to the KJT exactly; the dedup step's
outputs equal the KJT step's bit for bit (reference: dedup == baseline,
cli.py:284-289); the backward + SGD is deterministic; and one key is checked
against the oracle outright.  Tables are 1M x 128 per key (the properties do
not depend on the vocabulary)."""

import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu

import paper_2211_05239_b200 as R  # noqa: E402
from tools.datagen import SampleCountDist, SessionConfig, cfg2_specs, generate_clustered_batch  # noqa: E402,E501
from paper_2211_05239_b200.step import TrainStep  # noqa: E402

B, VOCAB, D = 65536, 1_000_000, 128


@pytest.fixture(scope="module")
def batch():
    return generate_clustered_batch(SessionConfig(B // 16, SampleCountDist("geometric", 16.5), 0),
                                    cfg2_specs(VOCAB), B)


def _tables(keys, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return {k: R.EmbeddingTable(k, VOCAB, D, torch.empty((VOCAB, D), device="cuda").uniform_(-0.1, 0.1,
                                                                                             generator=g))
            for k in keys}


def test_ikjt_round_trip_full_size(batch):
    keys = list(batch.keys)
    kjt = R.KJT(B, {k: R.JaggedTensor(batch.values[k], batch.offsets[k]) for k in keys})
    iks = R.kjt_to_ikjts(kjt, [[k] for k in keys])
    assert sum(int(kjt.entries[k].values.numel()) for k in keys) == 133_693_440
    for k, ik in zip(keys, iks):
        assert R.jt_equal(R.ikjt_to_kjt(ik).entries[k], kjt.entries[k]), k
    # one long-list key against the oracle outright
    k = keys[5]
    inv, [(uv, uo)] = oracle.build_ikjt_arrays([(batch.values[k], batch.offsets[k])])
    np.testing.assert_array_equal(iks[5].inverse_lookup.cpu().numpy(), inv)
    gv, go = iks[5].per_feature[k].numpy()
    np.testing.assert_array_equal(gv, uv)
    np.testing.assert_array_equal(go, uo)


def test_dedup_step_equals_kjt_step_and_is_deterministic(batch):
    keys = list(batch.keys)
    caps = {k: int(batch.values[k].size) for k in keys}
    outs, tabs = {}, {}
    for mode in ("dedup", "kjt", "dedup"):
        tables = _tables(keys, 7)
        step = TrainStep([[k] for k in keys], B, caps, tables, "sum", 0.05, mode)
        step.load_batch(batch.values, batch.offsets)
        step.fill_grad_out(3)
        step.run()
        torch.cuda.synchronize()
        o = [t.clone() for t in step.out]
        if mode in outs:   # second dedup run: bit-identical outputs and tables
            assert all(torch.equal(a, b) for a, b in zip(outs[mode], o))
            assert all(torch.equal(tabs[mode][k], tables[k].weights) for k in keys)
        else:
            outs[mode] = o
            tabs[mode] = {k: tables[k].weights.clone() for k in keys}
        del step, tables
        torch.cuda.empty_cache()
    # forward: the dedup path reproduces the KJT path bit for bit
    assert all(torch.equal(a, b) for a, b in zip(outs["dedup"], outs["kjt"]))
    # backward: the summation order differs (unique rows first), so the SGD updates
    # agree to the north_star tolerance (rtol 1e-5, atol 1e-5 * max |update|)
    w0 = _tables(keys, 7)
    for k in keys:
        u_d = w0[k].weights - tabs["dedup"][k]
        u_k = w0[k].weights - tabs["kjt"][k]
        scale = float(u_k.abs().max())
        assert scale > 0
        torch.testing.assert_close(u_d, u_k, rtol=1e-5, atol=1e-5 * scale)


def test_full_cfg2_against_oracle_touched_rows():
    """The bench's exact workload -- cfg2 B = 65,536, 26 keys, 26 tables of
    10M x 128 fp32 (133 GB on one B200) -- one TrainStep (dedup, pooled
    lookup, expand, backward + fused SGD), then for a length-8, a length-128
    and a length-256 key: IKJT, expanded pooled output and every SGD-updated
    table row bit-exact against the oracle (which sees only the touched rows:
    the unique IDs' rows, remapped into a compact table), untouched rows
    unchanged.  This exercises the 10M-row / 27M-unique-value code paths
    (32-bit chunk-relative positions, (f << 24) | u tags, 24-bit sort keys)."""
    rows, lr = 10_000_000, 0.05
    nsess = int(np.ceil(B / 16.5 * 1.3)) + 64       # bench.make_batch's session count
    b = generate_clustered_batch(SessionConfig(nsess, SampleCountDist("geometric", 16.5), 0),
                                 cfg2_specs(rows), B)
    keys = list(b.keys)
    tables = {k: R.EmbeddingTable.create_on_device(k, rows, D, seed=i) for i, k in enumerate(keys)}
    check = [0, 4, 5]       # list lengths 8, 128, 256
    w0 = {}
    for f in check:
        k = keys[f]
        inv, [(uv, uo)] = oracle.build_ikjt_arrays([(b.values[k], b.offsets[k])])
        ids = np.unique(uv)
        w0[k] = (inv, uv, uo, ids, tables[k].weights[torch.as_tensor(ids, device="cuda")].cpu().numpy())
    probe = torch.randint(0, rows, (4096,), device="cuda")
    before = {keys[f]: tables[keys[f]].weights[probe].clone() for f in check}
    caps = {k: int(b.values[k].size) for k in keys}
    step = TrainStep([[k] for k in keys], B, caps, tables, "sum", lr, "dedup")
    step.load_batch(b.values, b.offsets)
    step.fill_grad_out(11)
    step.run()
    torch.cuda.synchronize()
    step.check()
    for f in check:
        k = keys[f]
        inv, uv, uo, ids, wsub = w0[k]
        np.testing.assert_array_equal(step.inverse[f].cpu().numpy(), inv)
        U, NU = int(step.counts[f]), int(step.counts[len(keys) + f])
        assert (U, NU) == (uo.size, uv.size)
        np.testing.assert_array_equal(step.uoffsets[f][:U].cpu().numpy(), uo)
        np.testing.assert_array_equal(step.uvalues[f][:NU].cpu().numpy(), uv)
        loc = np.searchsorted(ids, uv)            # IDs -> rows of the compact table
        ref = oracle.expand(oracle.pooled_lookup(loc, uo, wsub, "sum"), inv)
        np.testing.assert_array_equal(step.out[f].cpu().numpy(), ref, err_msg=k)
        del ref
        G = step.grad_out[f].cpu().numpy()
        gu = oracle.pool_backward(G, inv, uo.size)
        lids, g = oracle.sparse_table_grad(gu, loc, uo, "sum")
        assert np.array_equal(lids, np.arange(ids.size))
        want = wsub - (np.float32(lr) * g).astype(np.float32)
        got = tables[k].weights[torch.as_tensor(ids, device="cuda")].cpu().numpy()
        np.testing.assert_array_equal(got, want, err_msg=k)
        untouched = ~torch.isin(probe, torch.as_tensor(ids, device="cuda"))
        assert torch.equal(tables[k].weights[probe][untouched], before[k][untouched])
    del step
    tables.clear()
    torch.cuda.empty_cache()
