"""jagged_index_select / ikjt_to_kjt / slice_ikjt_rows on the GPU vs golden."""

import json

import numpy as np
import pytest
import torch

import oracle
from conftest import dedup_cases, golden

pytestmark = pytest.mark.gpu

import paper_2211_05239_b200 as R  # noqa: E402


def test_jagged_index_select_matches_reference():
    g = golden("jagged")
    for c in range(int(g["count"][0])):
        jt = R.JaggedTensor(g[f"c{c}/values"], g[f"c{c}/offsets"])
        out = R.jagged_index_select(jt, g[f"c{c}/idx"])
        v, o = out.numpy()
        np.testing.assert_array_equal(v, g[f"c{c}/out_values"])
        np.testing.assert_array_equal(o, g[f"c{c}/out_offsets"])


def test_index_error_text():
    msgs = json.loads(str(golden("errors")["json"][0]))
    jt = R.JaggedTensor.from_rows([[1], [2]])
    with pytest.raises(IndexError) as e:
        R.jagged_index_select(jt, np.array([0, 5, -1]))
    assert str(e.value) == msgs["index_oob"][1]


def test_empty_selection():
    jt = R.JaggedTensor.from_rows([[1, 2]])
    out = R.jagged_index_select(jt, np.array([], dtype=np.int64))
    assert out.row_count == 0 and out.values.numel() == 0


def test_dense_pad_oracle_randomized():
    rng = np.random.default_rng(70)
    for _ in range(300):
        n_rows = int(rng.integers(1, 11))
        rows = [rng.integers(0, 100, size=rng.integers(0, 7)).tolist() for _ in range(n_rows)]
        jt = R.JaggedTensor.from_rows(rows)
        idx = rng.integers(0, n_rows, size=int(rng.integers(0, 17)))
        assert R.jagged_index_select(jt, idx).to_pylists() == [rows[i] for i in idx]


@pytest.mark.parametrize("case", list(dedup_cases())[::3], ids=lambda c: c[0])
def test_ikjt_to_kjt_round_trip(case):
    name, feats, inv_ref, outs_ref = case
    names = [f"f{i}" for i in range(len(feats))]
    kjt = R.KJT(len(feats[0][1]), {n: R.JaggedTensor(v, o) for n, (v, o) in zip(names, feats)})
    back = R.ikjt_to_kjt(R.kjt_to_ikjt(kjt, names))
    assert R.kjt_equal(back, kjt)


def test_slice_matches_reference():
    g = golden("slice")
    for c in range(int(g["count"][0])):
        per = {f"f{f}": R.JaggedTensor(g[f"c{c}/in{f}_values"], g[f"c{c}/in{f}_offsets"])
               for f in range(2)}
        inv = g[f"c{c}/inverse"]
        ik = R.IKJT(inv.size, ["f0", "f1"], inv, per)
        a, z = (int(x) for x in g[f"c{c}/range"])
        sub = R.slice_ikjt_rows(ik, a, z)
        np.testing.assert_array_equal(sub.inverse_lookup.cpu().numpy(), g[f"c{c}/out_inverse"])
        for f in range(2):
            v, o = sub.per_feature[f"f{f}"].numpy()
            np.testing.assert_array_equal(v, g[f"c{c}/out{f}_values"])
            np.testing.assert_array_equal(o, g[f"c{c}/out{f}_offsets"])


def test_split_equals_per_chunk_dedup():
    """slice_ikjt_rows == build_ikjt(rows[a:b]) (test_trainer_sim.py:391-398)."""
    rng = np.random.default_rng(4)
    b = 1001
    vals, offs, pos, state = [], [], 0, None
    for i in range(b):
        if state is None or rng.random() > 0.6:
            state = rng.integers(0, 9, size=int(rng.integers(0, 4)))
        offs.append(pos)
        vals.append(state)
        pos += state.size
    v, o = np.concatenate(vals).astype(np.int64), np.array(offs, np.int64)
    ik = R.kjt_to_ikjt(R.KJT(b, {"u": R.JaggedTensor(v, o)}), ["u"])
    start = 0
    for chunk in R.split_ikjt(ik, 4):
        stop = start + chunk.batch_size
        cv, co = oracle.jagged_index_select(v, o, np.arange(start, stop))
        inv, [(uv, uo)] = oracle.build_ikjt_arrays([(cv, co)])
        np.testing.assert_array_equal(chunk.inverse_lookup.cpu().numpy(), inv)
        got_v, got_o = chunk.per_feature["u"].numpy()
        np.testing.assert_array_equal(got_v, uv)
        np.testing.assert_array_equal(got_o, uo)
        start = stop
    with pytest.raises(ValueError):
        R.slice_ikjt_rows(ik, 0, b + 1)
