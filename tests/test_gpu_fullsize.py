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
