"""Partial (shift-aware) IKJT on the GPU (recd_partial_ikjt) vs the real
reference's build_partial_ikjt (tests/golden/partial.npz) and the oracle
restatement (oracle/partial.py): values and windows bit-exact.  At full size
(B = 65,536, rows up to 256 IDs) through the size-independent properties:
every window reconstructs its row, equal rows share a window, and the buffer
is no larger than the exact-dedup values."""

import numpy as np
import pytest
import torch

from conftest import golden

pytestmark = pytest.mark.gpu

import paper_2211_05239_b200 as R  # noqa: E402
from tools.datagen import (FeatureSpec, SampleCountDist, SessionConfig,  # noqa: E402
                                           generate_clustered_batch)


def _check(pk, values, windows, what):
    np.testing.assert_array_equal(pk.values.cpu().numpy(), values, err_msg=what)
    np.testing.assert_array_equal(pk.windows.cpu().numpy(), windows, err_msg=what)


def _kjt(values, offsets, key="f"):
    return R.KJT(offsets.size, {key: R.JaggedTensor(values, offsets)})


def test_partial_matches_reference_golden():
    d = golden("partial")
    for name in d["names"]:
        name = str(name)
        pk = R.kjt_to_partial_ikjt(_kjt(d[f"{name}/in_values"], d[f"{name}/in_offsets"]), "f")
        _check(pk, d[f"{name}/values"], d[f"{name}/windows"], name)


def test_partial_from_records_worked_example():
    """tests/test_acceptance.py:119-129 of the reference."""
    rows = [{"b": [3, 4, 5]}, {"b": [4, 5, 6]}, {"b": [3, 4, 5]}]
    pk = R.build_partial_ikjt(rows, "b")
    assert pk.values.cpu().tolist() == [3, 4, 5, 6]
    assert pk.windows.cpu().tolist() == [[0, 3], [1, 3], [0, 3]]
    assert pk.feature_key == "b" and pk.row_count == 3
    assert pk.row(1).cpu().tolist() == [4, 5, 6]
    assert pk.rounds == 1


def _random_case(seed, b, vocab, max_len, p_shift, mean_session):
    rng = np.random.default_rng(seed)
    lists = []
    while len(lists) < b:
        n = int(rng.integers(0, max_len + 1))
        count = 1 + int(rng.poisson(mean_session - 1))
        shifts = np.concatenate([[0], np.cumsum(rng.choice(3, size=count - 1, p=p_shift))])
        pool = rng.integers(-vocab // 4, vocab, size=n + int(shifts[-1]))
        lists += [pool[s:s + n] for s in shifts[: b - len(lists)]]
    lens = np.array([x.size for x in lists], dtype=np.int64)
    offsets = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.int64)
    values = np.concatenate(lists).astype(np.int64) if lens.sum() else np.empty(0, np.int64)
    return values, offsets


@pytest.mark.parametrize("seed,b,vocab,max_len,p_shift,mean", [
    (0, 4096, 1 << 40, 32, (0.5, 0.35, 0.15), 16.5),   # cfg1-like sessions
    (1, 3000, 10, 6, (0.3, 0.4, 0.3), 3.0),             # tiny vocab: found rows, deep overlaps
    (2, 2000, 3, 12, (0.2, 0.5, 0.3), 2.0),
    (3, 1, 100, 8, (1.0, 0.0, 0.0), 1.0),               # one row
    (4, 512, 1 << 62, 300, (0.1, 0.8, 0.1), 8.0),       # long rows
])
def test_partial_matches_oracle_random(seed, b, vocab, max_len, p_shift, mean):
    from oracle.partial import build_partial_jagged
    values, offsets = _random_case(seed, b, vocab, max_len, p_shift, mean)
    want_v, want_w = build_partial_jagged(values, offsets)
    pk = R.kjt_to_partial_ikjt(_kjt(values, offsets), "f")
    _check(pk, want_v, want_w, f"seed {seed}")


def test_partial_all_empty_rows():
    pk = R.kjt_to_partial_ikjt(_kjt(np.empty(0, np.int64), np.zeros(7, np.int64)), "f")
    assert pk.values.numel() == 0
    assert pk.windows.cpu().tolist() == [[0, 0]] * 7


def test_partial_empty_batch_and_validation():
    with pytest.raises(ValueError, match="empty batch"):
        R.build_partial_ikjt([], "f")
    with pytest.raises(ValueError, match="window exceeds value buffer"):
        R.PartialIKJT("b", [1, 2], [[1, 2]])
    with pytest.raises(ValueError, match="negative window bound"):
        R.PartialIKJT("b", [1, 2], [[-1, 1]])
    with pytest.raises(ValueError, match=r"\(B, 2\)"):
        R.PartialIKJT("b", [1, 2], [1, 2])


def test_partial_fullsize_properties():
    """cfg2's longest key (len 256) at B = 65,536, session-clustered."""
    B = 65536
    spec = FeatureSpec("hist", "user_sequence", 256.0, 10_000_000, 0.15)
    batch = generate_clustered_batch(SessionConfig(B // 8, SampleCountDist("geometric", 16.5), 3), [spec], B)
    kjt = R.KJT(B, {"hist": R.JaggedTensor(batch.values["hist"], batch.offsets["hist"])})
    ik = R.kjt_to_ikjt(kjt, ["hist"])
    pk = R.kjt_to_partial_ikjt(kjt, "hist", ik)
    jt = kjt.entries["hist"]
    lens = jt.row_lengths()
    win = pk.windows
    assert torch.equal(win[:, 1], lens)
    # every window reconstructs its row: values[win0[row] + j] == row[j]
    row_of = torch.repeat_interleave(torch.arange(B, device=lens.device), lens)
    j = torch.arange(jt.values.numel(), device=lens.device) - jt.offsets[row_of]
    assert torch.equal(pk.values[win[row_of, 0] + j], jt.values)
    # rows of one unique row share its window; the buffer is at most the unique values
    inv = ik.inverse_lookup
    first = torch.full((ik.unique_count,), B, dtype=torch.int64, device=inv.device)
    first.scatter_reduce_(0, inv, torch.arange(B, device=inv.device), "amin")
    assert torch.equal(win[:, 0], win[first[inv], 0])
    nu = ik.per_feature["hist"].values.numel()
    assert pk.values.numel() <= nu
    # shifted sessions: most unique rows append a single ID
    assert pk.values.numel() < 0.5 * nu
    assert pk.rounds <= 2
