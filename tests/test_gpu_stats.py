"""IterationStats from the CUDA dedup's device-side sizes (per-chunk
recd_dedup via kjt_to_ikjts, attention sequence lengths reduced on the GPU)
against the real reference's forward_iteration counters (tests/golden/sdd.npz)."""

import pytest
import torch

from conftest import golden

pytestmark = pytest.mark.gpu

import paper_2211_05239_b200 as R_  # noqa: E402
from paper_2211_05239_b200.stats import (chunk_sizes, ikjt_attention_macs,  # noqa: E402
                                         iteration_stats, split_bounds)
from test_stats import GROUPS, PLAIN, chunk  # noqa: E402


@pytest.mark.parametrize("R", [1, 2, 4, 8])
@pytest.mark.parametrize("mode", ["dedup", "baseline"])
def test_device_stats_match_reference(mode, R):
    d = golden("sdd")
    keys = [str(k) for k in d["rows/keys"]]
    dim = int(d["dim"][0])
    B = d[f"in/{keys[0]}/offsets"].size
    bounds = split_bounds(B, R)
    sizes, macs = [], {}
    for r, (a, b) in enumerate(bounds):
        ents = {}
        for k in keys:
            v, o = chunk(d[f"in/{k}/values"], d[f"in/{k}/offsets"], a, b)
            ents[k] = R_.JaggedTensor(torch.as_tensor(v).cuda(), torch.as_tensor(o).cuda())
        kjt = R_.KJT(b - a, ents)
        if mode == "dedup":
            iks = R_.kjt_to_ikjts(kjt, [g for g, _ in GROUPS])
        else:   # the baseline: identity inverse over the chunk's own rows
            iks = [R_.IKJT(b - a, g, torch.arange(b - a, device="cuda"),
                           {k: ents[k] for k in g}) for g, _ in GROUPS]
        plain = R_.KJT(b - a, {k: ents[k] for k in PLAIN})
        sizes.append(chunk_sizes(iks, plain))
        for gi, (g, pooling) in enumerate(GROUPS):
            if pooling == "attention":
                macs[(r, gi)] = ikjt_attention_macs(iks[gi], dim)
    st = iteration_stats(GROUPS, PLAIN, dim, sizes, [b - a for a, b in bounds], macs)
    assert st.as_list() == d[f"{mode}/R{R}/stats"].tolist()
