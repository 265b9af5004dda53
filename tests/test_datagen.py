"""The input generator restatement reproduces the reference generator's
batches bit for bit (checksums recorded from the real reference)."""

import hashlib

import numpy as np

from conftest import golden
from tools.datagen import (FeatureSpec, SampleCountDist, SessionConfig,
                                           cfg1_specs, generate_clustered_batch)


def _sha(v, o):
    return hashlib.sha256(np.ascontiguousarray(v).tobytes()
                          + np.ascontiguousarray(o).tobytes()).hexdigest()


def test_cfg1_batch_matches_reference_generator():
    g = golden("datagen")
    cfg = SessionConfig(600, SampleCountDist("geometric", 16.5), 0)
    b = generate_clustered_batch(cfg, cfg1_specs(), 4096)
    for k in b.keys:
        assert _sha(b.values[k], b.offsets[k]) == str(g[f"cfg1/{k}/sha"][0]), k
    np.testing.assert_array_equal(b.session_ids, g["cfg1/session_ids"])
    np.testing.assert_array_equal(b.labels, g["cfg1/labels"])


def test_mixed_kinds_match_reference_generator():
    g = golden("datagen")
    specs = [FeatureSpec("u", "user_sequence", 3.5, 50, 0.3, sync_group="g"),
             FeatureSpec("v", "user_sequence", 2.0, 50, 0.3, sync_group="g"),
             FeatureSpec("w", "user_sequence", 5.0, 1000, 0.5),
             FeatureSpec("it", "item", 2.5, 100)]
    cfg = SessionConfig(80, SampleCountDist("fixed", 8), 0)
    b = generate_clustered_batch(cfg, specs, 500)
    for k in b.keys:
        assert _sha(b.values[k], b.offsets[k]) == str(g[f"mixed/{k}/sha"][0]), k


def test_row_start_chunks_concatenate():
    cfg = SessionConfig(600, SampleCountDist("geometric", 16.5), 0)
    full = generate_clustered_batch(cfg, cfg1_specs()[:2], 1000)
    a = generate_clustered_batch(cfg, cfg1_specs()[:2], 400, row_start=0)
    z = generate_clustered_batch(cfg, cfg1_specs()[:2], 600, row_start=400)
    for k in full.keys:
        np.testing.assert_array_equal(np.concatenate([a.values[k], z.values[k]]), full.values[k])
