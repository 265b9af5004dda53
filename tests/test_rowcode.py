"""Row-delta coding of KJT rows for the H2D copy (librecd_host, CPU): the
host encoder against the host restatement of the device decode, on session
batches from the restated reference generator and on the edge cases (empty
rows, length changes, one-ID rows, rows that repeat an empty row, the first
row, literal capacity)."""

import numpy as np
import pytest

from paper_2211_05239_b200 import rowcode
from tools.datagen import FeatureSpec, SampleCountDist, SessionConfig, generate_clustered_batch


def _roundtrip(vals, offs, threads=0):
    B = offs[0].size
    codes = [np.full(B, 9, np.uint8) for _ in vals]
    lits = [np.empty(max(v.size, 1), np.int64) for v in vals]
    cnt = rowcode.encode(vals, offs, B, codes, lits, threads)
    for f, (v, o) in enumerate(zip(vals, offs)):
        assert set(np.unique(codes[f])) <= {rowcode.KEY, rowcode.REPEAT, rowcode.SHIFT}
        np.testing.assert_array_equal(rowcode.decode_reference(codes[f], o, v.size, lits[f][: cnt[f]]), v)
    return codes, cnt


@pytest.mark.parametrize("threads", [1, 3, 0])
def test_session_batch_round_trip(threads):
    specs = [FeatureSpec(f"k{i}", "user_sequence", float(L), 1000, 0.15) for i, L in enumerate([1, 4, 33, 256])]
    specs.append(FeatureSpec("item", "item", 5.5, 50))
    b = generate_clustered_batch(SessionConfig(300, SampleCountDist("geometric", 16.5), 7), specs, 4096)
    vals = [b.values[k] for k in b.keys]
    offs = [b.offsets[k] for k in b.keys]
    codes, cnt = _roundtrip(vals, offs, threads)
    # session rows repeat or shift: far fewer literals than values on the history keys
    assert cnt[3] * 8 < vals[3].size
    assert (codes[3] == rowcode.SHIFT).any() and (codes[3] == rowcode.REPEAT).any()


def test_edge_rows():
    rows = [[], [], [5], [5], [6], [1, 2, 3], [2, 3, 4], [2, 3, 4], [3, 4], [3, 4, 9], [4, 9, 9],
            [9, 9, 9], [9, 9, 9], [], [7], [7, 7], [7, 7]]
    offs = np.cumsum([0] + [len(r) for r in rows[:-1]]).astype(np.int64)
    vals = np.array([x for r in rows for x in r], dtype=np.int64)
    codes, cnt = _roundtrip([vals], [offs])
    c = codes[0]
    assert c[0] == rowcode.KEY and c[1] == rowcode.REPEAT      # empty after empty
    assert c[3] == rowcode.REPEAT and c[4] == rowcode.SHIFT    # one-ID rows
    assert c[6] == rowcode.SHIFT and c[7] == rowcode.REPEAT and c[8] == rowcode.KEY  # length change


def test_random_rows_and_capacity():
    rng = np.random.default_rng(3)
    for _ in range(5):
        B = int(rng.integers(1, 400))
        lens = rng.integers(0, 6, size=B)
        vals = rng.integers(0, 3, size=int(lens.sum())).astype(np.int64)   # tiny vocab: many matches
        offs = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.int64)
        _roundtrip([vals], [offs], threads=int(rng.integers(0, 4)))
    vals = np.arange(10, dtype=np.int64)
    offs = np.array([0, 5], dtype=np.int64)
    with pytest.raises(ValueError, match="capacity"):
        rowcode.encode([vals], [offs], 2, [np.empty(2, np.uint8)], [np.empty(4, np.int64)])


def test_raw_key_share_met_from_below():
    """H2DPipeline copies the largest keys raw up to raw_share of the IDs,
    skipping a key that would overshoot (cfg2: 4 keys of 256 IDs per row are
    12.6% each, so 0.28 takes two of them plus shorter keys, not three)."""
    import types

    from paper_2211_05239_b200.staging import H2DPipeline

    n = [L * 1000 for L in ([8, 16, 32, 64, 128, 256] * 5)[:26]]
    pick = lambda share: H2DPipeline._raw_keys(types.SimpleNamespace(raw_share=share), n)
    tot = sum(n)
    for share in (0.0, 0.1, 0.2, 0.28, 0.5, 1.0):
        raw = pick(share)
        got = sum(n[f] for f in raw)
        assert got <= share * tot
        # nothing left out that would still fit
        assert all(n[f] == 0 or got + n[f] > share * tot for f in range(len(n)) if f not in raw)
    assert sorted(n[f] for f in pick(0.28)).count(256000) == 2
    assert pick(1.0) == set(range(len(n)))
