"""Pin the CPU oracle against golden vectors produced by the real reference.

These run without a GPU (`-m "not gpu"`).  If the oracle drifted from the
reference, every GPU parity claim built on it would be void.
"""

import json

import numpy as np
import pytest

import oracle
from conftest import dedup_cases, golden


@pytest.mark.parametrize("case", list(dedup_cases()), ids=lambda c: c[0])
def test_oracle_dedup_matches_reference(case):
    name, feats, inv_ref, outs_ref = case
    inv, outs = oracle.build_ikjt_arrays(feats)
    np.testing.assert_array_equal(inv, inv_ref)
    for (uv, uo), (rv, ro) in zip(outs, outs_ref):
        np.testing.assert_array_equal(uv, rv)
        np.testing.assert_array_equal(uo, ro)
    # expansion invariant (tensors.py:393-399, SPEC round-trip property)
    for (v, o), (xv, xo) in zip(feats, oracle.ikjt_to_kjt_arrays(inv, outs)):
        np.testing.assert_array_equal(xv, v)
        np.testing.assert_array_equal(xo, o)


def test_oracle_cfg1_dedup_matches_reference():
    from tools.datagen import (SampleCountDist, SessionConfig, cfg1_specs,
                                               generate_clustered_batch)
    g = golden("datagen")
    cfg = SessionConfig(600, SampleCountDist("geometric", 16.5), 0)
    batch = generate_clustered_batch(cfg, cfg1_specs(), 4096)
    for k in batch.keys:
        inv, [(uv, uo)] = oracle.build_ikjt_arrays([(batch.values[k], batch.offsets[k])])
        np.testing.assert_array_equal(inv, g[f"cfg1/{k}/inverse"])
        np.testing.assert_array_equal(uv, g[f"cfg1/{k}/uvalues"])
        np.testing.assert_array_equal(uo, g[f"cfg1/{k}/uoffsets"])


@pytest.mark.parametrize("dim", [1, 4, 8, 64, 128])
@pytest.mark.parametrize("op", ["sum", "avg", "max"])
def test_oracle_pool_matches_reference(dim, op):
    g = golden("pool")
    w = g[f"d{dim}/weights"]
    pooled = oracle.pooled_lookup(g[f"d{dim}/values"], g[f"d{dim}/offsets"], w, op)
    np.testing.assert_array_equal(pooled, g[f"d{dim}/{op}"])  # bit-exact
    np.testing.assert_array_equal(oracle.expand(pooled, g[f"d{dim}/inverse"]),
                                  g[f"d{dim}/{op}_expanded"])


def test_oracle_jagged_index_select_matches_reference():
    g = golden("jagged")
    for c in range(int(g["count"][0])):
        v, o = oracle.jagged_index_select(g[f"c{c}/values"], g[f"c{c}/offsets"], g[f"c{c}/idx"])
        np.testing.assert_array_equal(v, g[f"c{c}/out_values"])
        np.testing.assert_array_equal(o, g[f"c{c}/out_offsets"])


def test_oracle_slice_matches_reference():
    g = golden("slice")
    for c in range(int(g["count"][0])):
        feats = [(g[f"c{c}/in{f}_values"], g[f"c{c}/in{f}_offsets"]) for f in range(2)]
        a, z = (int(x) for x in g[f"c{c}/range"])
        inv, outs = oracle.slice_ikjt_rows(g[f"c{c}/inverse"], feats, a, z)
        np.testing.assert_array_equal(inv, g[f"c{c}/out_inverse"])
        for f, (v, o) in enumerate(outs):
            np.testing.assert_array_equal(v, g[f"c{c}/out{f}_values"])
            np.testing.assert_array_equal(o, g[f"c{c}/out{f}_offsets"])


def test_oracle_error_messages_match_reference():
    msgs = json.loads(str(golden("errors")["json"][0]))
    with pytest.raises(ValueError) as e:
        oracle.build_ikjt_rows([], ["a"])
    assert str(e.value) == msgs["empty_batch"][1]
    with pytest.raises(ValueError) as e:
        oracle.build_ikjt_rows([{"a": [1]}], [])
    assert str(e.value) == msgs["empty_group"][1]
    with pytest.raises(IndexError) as e:
        oracle.jagged_index_select(np.array([1, 2]), np.array([0, 1]), np.array([0, 5, -1]))
    assert str(e.value) == msgs["index_oob"][1]
    w = np.arange(4, dtype=np.float32).reshape(-1, 1)
    with pytest.raises(ValueError) as e:
        oracle.embedding_lookup(np.array([1, 9, 3]), w, "b")
    assert str(e.value) == msgs["id_oob"][1]
    with pytest.raises(ValueError) as e:
        oracle.pool(np.zeros((1, 1), dtype=np.float32), np.array([0]), "median")
    assert str(e.value) == msgs["pool_op"][1]


def test_transforms_oracle_matches_reference_golden():
    """reader.apply_transform (reader.py:69-83) restated in oracle/reader.py."""
    d = golden("transforms")
    v = d["values"]
    for i in range(int(d["ncases"][0])):
        op, param = str(d[f"c{i}/op"][0]), int(d[f"c{i}/param"][0])
        got = oracle.apply_transform(v, op, param or None)
        np.testing.assert_array_equal(got, d[f"c{i}/out"])


def test_wire_oracle_matches_reference_golden():
    """tensors.serialize_kjt / serialize_ikjt (tensors.py:463-515) restated in oracle/wire.py."""
    d = golden("wire")
    for name in d["names"]:
        name = str(name)
        keys = [str(k) for k in d[f"{name}/keys"]]
        feats = [(d[f"{name}/in_{k}_values"], d[f"{name}/in_{k}_offsets"]) for k in keys]
        B = feats[0][1].size
        kjt = oracle.wire.serialize(keys, B, None, [o for _, o in feats], [v for v, _ in feats])
        assert kjt == d[f"{name}/kjt_bytes"].tobytes()
        inv, outs = oracle.build_ikjt_arrays(feats)
        ik = oracle.wire.serialize(keys, B, inv, [o for _, o in outs], [v for v, _ in outs])
        assert ik == d[f"{name}/ikjt_bytes"].tobytes()
        assert [oracle.wire.slice_stream_bytes(o, v) for v, o in outs] == list(d[f"{name}/slice_bytes"])
        assert [oracle.wire.values_stream_bytes(v) for v, _ in outs] == list(d[f"{name}/values_bytes"])


def test_partial_oracle_matches_reference_golden():
    """oracle/partial.py vs the real build_partial_ikjt (tests/golden/partial.npz):
    worked examples, found substrings, overlaps deeper than the previous row,
    int64 extremes, adversarial small vocabularies, session batches."""
    from oracle.partial import build_partial_jagged
    d = golden("partial")
    for name in d["names"]:
        name = str(name)
        v, w = build_partial_jagged(d[f"{name}/in_values"], d[f"{name}/in_offsets"])
        np.testing.assert_array_equal(v, d[f"{name}/values"], err_msg=name)
        np.testing.assert_array_equal(w, d[f"{name}/windows"], err_msg=name)


def test_partial_oracle_empty_batch():
    from oracle.partial import build_partial
    with pytest.raises(ValueError, match="empty batch"):
        build_partial([])
