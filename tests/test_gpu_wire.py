"""Canonical wire format assembled on the GPU vs the bytes of the real
reference's serialize_kjt / serialize_ikjt (tests/golden/wire.npz), incl.
UTF-8 key names, empty lists and unaligned section offsets."""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu

import paper_2211_05239_b200 as R  # noqa: E402


def test_wire_bytes_match_reference():
    d = golden("wire")
    for name in d["names"]:
        name = str(name)
        keys = [str(k) for k in d[f"{name}/keys"]]
        B = d[f"{name}/in_{keys[0]}_offsets"].size
        kjt = R.KJT(B, {k: R.JaggedTensor(d[f"{name}/in_{k}_values"], d[f"{name}/in_{k}_offsets"])
                        for k in keys})
        assert R.serialize_kjt(kjt) == d[f"{name}/kjt_bytes"].tobytes(), name
        ik = R.kjt_to_ikjt(kjt, keys)
        assert R.serialize_ikjt(ik) == d[f"{name}/ikjt_bytes"].tobytes(), name
        assert [R.slice_stream_bytes(ik.per_feature[k]) for k in keys] == list(d[f"{name}/slice_bytes"])
        assert [R.values_stream_bytes(ik.per_feature[k]) for k in keys] == list(d[f"{name}/values_bytes"])


@pytest.mark.parametrize("klen", [1, 2, 3, 5, 7, 8])
def test_wire_all_alignments(klen):
    """Key-name lengths shift every section to each byte alignment."""
    import oracle
    rng = np.random.default_rng(klen)
    key = "k" * klen
    b = 257
    lens = rng.integers(0, 9, size=b)
    v = rng.integers(-2**62, 2**62, size=int(lens.sum()), dtype=np.int64)
    o = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.int64)
    kjt = R.KJT(b, {key: R.JaggedTensor(v, o)})
    assert R.serialize_kjt(kjt) == oracle.wire.serialize([key], b, None, [o], [v])
