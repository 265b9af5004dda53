"""Native host-side KJT packing (csrc/host/recd_hostpack.cpp) against the
oracle's build_kjt restatement (tensors.py:228-254): dict rows, objects with
`.features`, absent keys, numpy lists, error texts.  CPU only."""

from types import SimpleNamespace

import numpy as np
import pytest

import oracle


@pytest.fixture(scope="module")
def hostpack():
    from paper_2211_05239_b200.build import build_host
    build_host()
    from paper_2211_05239_b200 import _hostpack
    return _hostpack


def _unpack(packed):
    return [(np.frombuffer(v, np.int64), np.frombuffer(o, np.int64)) for v, o in packed]


def test_pack_matches_oracle(hostpack):
    rng = np.random.default_rng(0)
    keys = ["a", "b", "c"]
    rows = []
    for i in range(500):
        r = {k: rng.integers(-2**62, 2**62, size=int(rng.integers(0, 12))).tolist()
             for k in keys if rng.random() < 0.8}
        if i % 7 == 0:
            r["a"] = np.array(r.get("a", []), dtype=np.int64)       # numpy lists
        rows.append(r if i % 5 else SimpleNamespace(features=r))   # objects with .features
    got = _unpack(hostpack.pack_rows(rows, keys))
    ref = oracle.build_kjt_arrays(rows, keys)
    for k, (v, o) in zip(keys, got):
        np.testing.assert_array_equal(v, ref[k][0])
        np.testing.assert_array_equal(o, ref[k][1])


def test_pack_errors(hostpack):
    with pytest.raises(ValueError, match="one-dimensional"):
        hostpack.pack_rows([{"a": [[1, 2]]}], ["a"])
    with pytest.raises(TypeError, match="cannot extract features from int"):
        hostpack.pack_rows([3], ["a"])
    with pytest.raises(OverflowError):
        hostpack.pack_rows([{"a": [2**64]}], ["a"])


def test_pack_converter_matches_reference_semantics(hostpack):
    """Inputs off the fast path go through the reference's conversion
    (np.asarray(dtype=int64) + 1-D check, tensors.py:47-51)."""
    from paper_2211_05239_b200.tensors import _as_id_array
    rows = [{"a": [1.9, 2.2]}, {"a": np.array([[3], [4]]).ravel()}, {"a": (5, np.int32(6))},
            {"a": np.arange(3, dtype=np.uint8)}]
    got = _unpack(hostpack.pack_rows(rows, ["a"], _as_id_array))
    ref = oracle.build_kjt_arrays(rows, ["a"])
    np.testing.assert_array_equal(got[0][0], ref["a"][0])
    np.testing.assert_array_equal(got[0][1], ref["a"][1])
    with pytest.raises(ValueError, match=r"one-dimensional, got shape \(\)"):
        hostpack.pack_rows([{"a": 7}], ["a"], _as_id_array)
    with pytest.raises(ValueError, match=r"one-dimensional, got shape \(1, 2\)"):
        hostpack.pack_rows([{"a": [[1, 2]]}], ["a"], _as_id_array)
    with pytest.raises(ValueError, match=r"one-dimensional, got shape \(2, 1\)"):
        hostpack.pack_rows([{"a": np.zeros((2, 1), np.int64)}], ["a"], _as_id_array)
