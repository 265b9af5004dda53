"""Reader transforms on the GPU (reader.py:54-83, 178-217) against the golden
vectors of the real reference, and the dedup property: transforming an
IKJT's unique values then expanding equals transforming the KJT
(test_reader.py:176-187)."""

import numpy as np
import pytest
import torch

from conftest import golden

pytestmark = pytest.mark.gpu

import paper_2211_05239_b200 as R  # noqa: E402
from paper_2211_05239_b200.reader import (DataloaderSpec, Transform, apply_transform, convert,  # noqa: E402
                                          process, process_tensors)


def test_transforms_match_reference_golden():
    d = golden("transforms")
    v = torch.as_tensor(d["values"], device="cuda")
    for i in range(int(d["ncases"][0])):
        op, param = str(d[f"c{i}/op"][0]), int(d[f"c{i}/param"][0])
        out = apply_transform(v, Transform(op, "k", param or None))
        np.testing.assert_array_equal(out.cpu().numpy(), d[f"c{i}/out"])


def test_transform_errors_like_reference():
    with pytest.raises(ValueError, match="unknown transform op 'hash'"):
        Transform("hash", "k", 3)
    with pytest.raises(ValueError, match="mod_hash needs a positive param"):
        Transform("mod_hash", "k", 0)
    kjt = R.KJT(2, {"a": R.JaggedTensor(np.array([1, 2], np.int64), np.array([0, 1], np.int64))})
    with pytest.raises(ValueError, match="transform targets missing key 'zz'"):
        process_tensors(kjt.entries, [], [Transform("clamp", "zz", 3)])


def test_transform_commutes_with_expansion():
    rng = np.random.default_rng(2)
    b = 3000
    vals, offs, pos, state = [], [], 0, None
    for i in range(b):
        if state is None or rng.random() > 0.8:
            state = rng.integers(0, 1 << 40, size=int(rng.integers(0, 20)))
        offs.append(pos)
        vals.append(state)
        pos += state.size
    v, o = np.concatenate(vals).astype(np.int64), np.array(offs, np.int64)
    kjt = R.KJT(b, {"h": R.JaggedTensor(v, o), "p": R.JaggedTensor(v[::-1].copy(), o)})
    ik = R.kjt_to_ikjt(kjt, ["h"])
    ts = [Transform("mod_hash", "h", 1_000_003), Transform("clamp", "h", 500_000),
          Transform("mod_hash", "p", 97)]
    plain, [ik2] = process_tensors({"p": kjt.entries["p"]}, [ik], ts)
    expanded = R.ikjt_to_kjt(ik2).entries["h"]
    ref_h, _ = process_tensors({"h": kjt.entries["h"]}, [], ts[:2])
    assert R.jt_equal(expanded, ref_h["h"])
    assert torch.equal(ik2.inverse_lookup, ik.inverse_lookup)
    ref_p = apply_transform(kjt.entries["p"], ts[2])
    assert R.jt_equal(plain["p"], ref_p)


def test_reader_convert_process_like_reference():
    """reader.convert + reader.process (reader.py:160-217) on records with
    labels: groups become IKJTs equal to build_ikjt, plain keys stay jagged,
    transforms hit unique values only."""
    import oracle
    from types import SimpleNamespace
    rng = np.random.default_rng(9)
    rows, state = [], None
    for i in range(700):
        if state is None or rng.random() > 0.8:
            state = {k: rng.integers(0, 1000, size=int(rng.integers(0, 9))).tolist() for k in ("a", "b", "c")}
        rows.append(SimpleNamespace(features=dict(state), label=i % 2))
    spec = DataloaderSpec(keys=("a", "b", "c"), dedup_sparse_features=(("a", "b"),),
                          transforms=(Transform("mod_hash", "a", 97),))
    batch = convert(rows, spec)
    assert batch.all_keys() == ("c", "a", "b")
    np.testing.assert_array_equal(batch.labels, np.arange(700) % 2)
    feats = [(np.array(sum([r.features["a"] for r in rows], []), np.int64),
              np.cumsum([0] + [len(r.features["a"]) for r in rows[:-1]]).astype(np.int64)),
             (np.array(sum([r.features["b"] for r in rows], []), np.int64),
              np.cumsum([0] + [len(r.features["b"]) for r in rows[:-1]]).astype(np.int64))]
    inv, outs = oracle.build_ikjt_arrays(feats)
    np.testing.assert_array_equal(batch.ikjts[0].inverse_lookup.cpu().numpy(), inv)
    out = process(batch, spec.transforms)
    v, _ = out.ikjts[0].per_feature["a"].numpy()
    np.testing.assert_array_equal(v, oracle.apply_transform(outs[0][0], "mod_hash", 97))
    with pytest.raises(ValueError, match="feature 'a' in more than one dedup group"):
        DataloaderSpec(keys=("a", "b"), dedup_sparse_features=(("a",), ("a", "b")))
