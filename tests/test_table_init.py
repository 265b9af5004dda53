"""EmbeddingTable.create reproduces the reference's seeded table init
(trainer_sim.py:62-66, 83-87) bit for bit: weights recorded from the real
`EmbeddingTable.create("k0", rows=64, dim=8, seed=0)` (tests/golden/datagen.npz)."""

import numpy as np
import pytest

from conftest import golden
from paper_2211_05239_b200.embedding import EmbeddingTable


def test_init_weights_match_reference():
    g = golden("datagen")
    w = EmbeddingTable.init_weights("k0", 64, 8, 0)
    assert w.dtype == np.float32
    np.testing.assert_array_equal(w, g["table_k0_64x8"])
    # other keys / seeds draw other streams
    assert not np.array_equal(EmbeddingTable.init_weights("k1", 64, 8, 0), w)
    assert not np.array_equal(EmbeddingTable.init_weights("k0", 64, 8, 1), w)


@pytest.mark.gpu
def test_create_on_gpu_matches_reference():
    import torch
    g = golden("datagen")
    t = EmbeddingTable.create("k0", 64, 8, 0, device=torch.device("cuda"))
    assert t.weights.is_cuda
    np.testing.assert_array_equal(t.weights.cpu().numpy(), g["table_k0_64x8"])
