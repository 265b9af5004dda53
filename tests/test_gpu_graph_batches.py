"""One captured CUDA graph for every batch: TrainStep(slots=2) is captured
once and then fed 20 distinct session batches through the H2D pipeline --
non-integer average lengths (per-session length draws) and an `item` key
(per-row lengths), so every batch has different value counts -- each step
bit-exact against the oracle, with the tables carried from step to step
(the reference's convert takes any batch, reader.py:160-175)."""

import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu

import paper_2211_05239_b200 as R  # noqa: E402
from paper_2211_05239_b200.staging import H2DPipeline  # noqa: E402
from paper_2211_05239_b200.step import TrainStep  # noqa: E402
from tools.datagen import FeatureSpec, SampleCountDist, SessionConfig, generate_clustered_batch  # noqa: E402

SPECS = [FeatureSpec("hist_a", "user_sequence", 7.4, 4000, 0.2),
         FeatureSpec("hist_b", "user_sequence", 23.6, 4000, 0.1),
         FeatureSpec("item", "item", 2.5, 4000)]


def _batches(n, b):
    return [generate_clustered_batch(SessionConfig(b // 4, SampleCountDist("geometric", 12.0), seed),
                                     SPECS, b) for seed in range(n)]


@pytest.mark.parametrize("mode,fused,wire", [("dedup", "0", "raw"), ("dedup", "1", "raw"),
                                             ("kjt", "0", "raw"), ("dedup", "1", "rowcode"),
                                             ("kjt", "0", "rowcode"), ("dedup", "1", "mixed")])
def test_one_graph_twenty_batches(mode, fused, wire, monkeypatch):
    """wire: raw int64 KJT copies, row-delta coded batches decoded on the
    device (H2DPipeline(rowcode=True)), or half the IDs raw and half coded."""
    monkeypatch.setenv("RECD_FUSED_EXPAND", fused)
    b, vocab, dim, lr = 1024, 4000, 32, 0.05
    batches = _batches(20, b)
    keys = [s.key for s in SPECS]
    sizes = {k: [x.values[k].size for x in batches] for k in keys}
    assert all(len(set(v)) > 5 for v in sizes.values()), sizes   # the counts really vary
    caps = {k: max(v) for k, v in sizes.items()}
    rng = np.random.default_rng(0)
    w = {k: rng.uniform(-0.1, 0.1, size=(vocab, dim)).astype(np.float32) for k in keys}
    tables = {k: R.EmbeddingTable(k, vocab, dim, torch.as_tensor(w[k], device="cuda").clone())
              for k in keys}
    grads = {k: rng.standard_normal((b, dim)).astype(np.float32) for k in keys}
    step = TrainStep([[k] for k in keys], b, caps, tables, "sum", lr, mode, slots=2)
    for f, k in enumerate(keys):
        step.grad_out[f].copy_(torch.as_tensor(grads[k]))
    # capture on a throw-away batch, then restore the tables
    step.load_batch(batches[0].values, batches[0].offsets, slot=0)
    step.load_batch(batches[0].values, batches[0].offsets, slot=1)
    step.capture()
    torch.cuda.synchronize()
    for k in keys:
        tables[k].weights.copy_(torch.as_tensor(w[k]))
    graphs = list(step.graphs)
    pipe = H2DPipeline(step, rowcode=wire != "raw", raw_share=0.5 if wire == "mixed" else 0.0)
    pin = [({k: torch.from_numpy(x.values[k]).pin_memory() for k in keys},
            {k: torch.from_numpy(x.offsets[k]).pin_memory() for k in keys}) for x in batches]
    pipe.prefetch(0, *pin[0])
    for i, x in enumerate(batches):
        if i + 1 < len(batches):
            pipe.prefetch((i + 1) % 2, *pin[i + 1])
        pipe.run(i % 2, step.replay)
        torch.cuda.synchronize()
        step.check()
        assert step.graphs == graphs            # never re-captured
        for f, k in enumerate(keys):
            v, o = x.values[k], x.offsets[k]
            if mode == "dedup":
                inv, [(uv, uo)] = oracle.build_ikjt_arrays([(v, o)])
            else:
                inv, uv, uo = np.arange(b), v, o
            ref = oracle.expand(oracle.pooled_lookup(uv, uo, w[k], "sum"), inv)
            np.testing.assert_array_equal(step.out[f].cpu().numpy(), ref, err_msg=f"batch {i} {k}")
            gu = oracle.pool_backward(grads[k], inv, uo.size)
            ids, g = oracle.sparse_table_grad(gu, uv, uo, "sum")
            w[k][ids] = w[k][ids] - (np.float32(lr) * g).astype(np.float32)
            np.testing.assert_array_equal(tables[k].weights.cpu().numpy(), w[k],
                                          err_msg=f"batch {i} {k}")


@pytest.mark.parametrize("mode", ["dedup", "kjt"])
def test_pipelined_step_matches_oracle(mode):
    """TrainStep(pipeline=True): graph i trains batch i while its side stream
    deduplicates batch i+1 (and sorts its occurrences); batches arrive through
    the H2D pipeline.  Every batch's outputs and table updates stay bit-exact
    against the sequential oracle."""
    b, vocab, dim, lr, n = 1024, 4000, 32, 0.05, 12
    batches = _batches(n + 1, b)
    keys = [s.key for s in SPECS]
    caps = {k: max(x.values[k].size for x in batches) for k in keys}
    rng = np.random.default_rng(1)
    w = {k: rng.uniform(-0.1, 0.1, size=(vocab, dim)).astype(np.float32) for k in keys}
    tables = {k: R.EmbeddingTable(k, vocab, dim, torch.as_tensor(w[k], device="cuda").clone())
              for k in keys}
    grads = {k: rng.standard_normal((b, dim)).astype(np.float32) for k in keys}
    step = TrainStep([[k] for k in keys], b, caps, tables, "sum", lr, mode, pipeline=True)
    for f, k in enumerate(keys):
        step.grad_out[f].copy_(torch.as_tensor(grads[k]))
    for s in range(2):
        step.load_batch(batches[0].values, batches[0].offsets, slot=s)
    step.capture()
    torch.cuda.synchronize()
    for k in keys:
        tables[k].weights.copy_(torch.as_tensor(w[k]))
    pipe = H2DPipeline(step)
    pin = [({k: torch.from_numpy(x.values[k]).pin_memory() for k in keys},
            {k: torch.from_numpy(x.offsets[k]).pin_memory() for k in keys}) for x in batches]
    pipe.prefetch(0, *pin[0])
    pipe.prefetch(1, *pin[1])
    pipe.wait_ready(0)
    step.prime(0)
    for i in range(n):
        p = i % 2
        pipe.wait_ready(1 - p)
        pipe.release(p)
        step.replay(p)
        if i + 2 <= n:
            pipe.prefetch(p, *pin[i + 2])
        torch.cuda.synchronize()
        step.check()
        x = batches[i]
        for f, k in enumerate(keys):
            v, o = x.values[k], x.offsets[k]
            if mode == "dedup":
                inv, [(uv, uo)] = oracle.build_ikjt_arrays([(v, o)])
            else:
                inv, uv, uo = np.arange(b), v, o
            ref = oracle.expand(oracle.pooled_lookup(uv, uo, w[k], "sum"), inv)
            np.testing.assert_array_equal(step.out[f].cpu().numpy(), ref, err_msg=f"batch {i} {k}")
            gu = oracle.pool_backward(grads[k], inv, uo.size)
            ids, g = oracle.sparse_table_grad(gu, uv, uo, "sum")
            w[k][ids] = w[k][ids] - (np.float32(lr) * g).astype(np.float32)
            np.testing.assert_array_equal(tables[k].weights.cpu().numpy(), w[k],
                                          err_msg=f"batch {i} {k}")
