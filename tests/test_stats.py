"""IterationStats (paper_2211_05239_b200/stats.py) against the real
reference's forward_iteration counters (tests/golden/sdd.npz, made by
tests/golden/make_golden.py from trainer_sim.py:484-586): sdd all-to-all
bytes, pooled rows back, lookups, activation peak, pooling MACs and
index-select elements at R in {1, 2, 4, 8} ranks, dedup and baseline.  The
per-chunk IKJT sizes come from the oracle here (CPU); test_gpu_stats.py
takes them from the CUDA dedup."""

import numpy as np
import pytest

import oracle
from conftest import golden
from paper_2211_05239_b200.stats import (STAT_FIELDS, IterationStats, attention_macs,
                                         iteration_stats, round_robin_plan, split_bounds)

GROUPS = [(("u", "v"), "attention"), (("w",), "sum"), (("x",), "avg"), (("y",), "max")]
PLAIN = {"it": "sum"}


def chunk(v, o, a, b):
    lo = int(o[a])
    hi = int(o[b]) if b < o.size else v.size
    return v[lo:hi], o[a:b] - lo


def oracle_sizes(d, mode, R):
    keys = [str(k) for k in d["rows/keys"]]
    dim = int(d["dim"][0])
    B = d[f"in/{keys[0]}/offsets"].size
    bounds = split_bounds(B, R)
    sizes, macs = [], {}
    for r, (a, b) in enumerate(bounds):
        sz = {}
        for gi, (gkeys, pooling) in enumerate(GROUPS):
            feats = [chunk(d[f"in/{k}/values"], d[f"in/{k}/offsets"], a, b) for k in gkeys]
            if mode == "dedup":
                _, outs = oracle.build_ikjt_arrays(feats)
            else:
                outs = feats
            lens = []
            for k, (uv, uo) in zip(gkeys, outs):
                sz[k] = (uo.size, uv.size)
                lens.append(np.diff(np.append(uo, uv.size)))
            if pooling == "attention":
                macs[(r, gi)] = attention_macs(lens, dim)
        for k in PLAIN:
            v, o = chunk(d[f"in/{k}/values"], d[f"in/{k}/offsets"], a, b)
            sz[k] = (o.size, v.size)
        sizes.append(sz)
    return sizes, [b - a for a, b in bounds], macs, dim


@pytest.mark.parametrize("R", [1, 2, 4, 8])
@pytest.mark.parametrize("mode", ["dedup", "baseline"])
def test_stats_match_reference(mode, R):
    d = golden("sdd")
    assert tuple(str(f) for f in d["fields"]) == STAT_FIELDS
    sizes, bs, macs, dim = oracle_sizes(d, mode, R)
    st = iteration_stats(GROUPS, PLAIN, dim, sizes, bs, macs)
    assert st.as_list() == d[f"{mode}/R{R}/stats"].tolist()


@pytest.mark.parametrize("R", [1, 2, 4, 8])
def test_plan_and_dominance(R):
    d = golden("sdd")
    keys = [str(k) for k in d["rows/keys"]]
    plan = round_robin_plan([g for g, _ in GROUPS], list(PLAIN), R)
    assert [plan[k] for k in keys] == d[f"dedup/R{R}/plan"].tolist()
    ded = IterationStats(*d[f"dedup/R{R}/stats"].tolist())
    base = IterationStats(*d[f"baseline/R{R}/stats"].tolist())
    assert ded.dominated_by(base) and not base.dominated_by(ded)


def test_split_bounds_matches_split_batch():
    assert split_bounds(10, 3) == [(0, 4), (4, 7), (7, 10)]
    with pytest.raises(ValueError):
        split_bounds(2, 3)
