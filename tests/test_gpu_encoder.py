"""Config 4: dedup'd sequence encoder (attention_pool over unique rows,
trainer_sim.py:347-391) against the fp32 oracle, and the tcgen05 BF16 GEMM
it is built on against torch.

Tolerances: the GEMM output is BF16 (FP32 accumulation), so it is compared
with an FP32 torch matmul of the same BF16 operands to 1 BF16 ulp
(rtol 2^-7).  The encoder uses BF16 operands for the QKV projection and the
scores, FP32 everywhere else; against the all-FP32 oracle the stated
tolerance is allclose(rtol=3e-2, atol=3e-2 * max|ref|).  Dedup vs KJT path:
the same rows go through the same kernels, so outputs are bit-identical (the
reference asserts dedup == baseline scores, cli.py:284-289)."""

import ctypes as C

import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu

import paper_2211_05239_b200 as R  # noqa: E402
from paper_2211_05239_b200 import _lib  # noqa: E402


@pytest.mark.parametrize("n,k,m", [(384, 128, 1000), (192, 64, 129), (128, 128, 4096), (384, 128, 1)])
def test_tcgen05_gemm_matches_torch(n, k, m):
    torch.manual_seed(n + k + m)
    a = torch.randn(m, k, device="cuda").to(torch.bfloat16)
    b = torch.randn(n, k, device="cuda").to(torch.bfloat16)
    c = torch.full((m, n), float("nan"), device="cuda").to(torch.bfloat16)
    mc = torch.tensor([m], dtype=torch.int64, device="cuda")
    rc = _lib.load().recd_gemm_bf16_tn(n, k, a.data_ptr(), b.data_ptr(), c.data_ptr(), mc.data_ptr(),
                                       _lib.stream_ptr())
    assert rc == 0
    torch.cuda.synchronize()
    ref = a.float() @ b.float().t()
    torch.testing.assert_close(c.float(), ref, rtol=2 ** -7, atol=1e-3)


def _grouped_batch(rng, b, vocab, lens, dup=0.8):
    """Synced group (datagen sync_group): all keys of a row change together."""
    vals = {k: [] for k in lens}
    offs = {k: [] for k in lens}
    pos = {k: 0 for k in lens}
    state = None
    for i in range(b):
        if state is None or rng.random() > dup:
            empty = rng.random() < 0.1   # some rows with no history at all
            state = {k: rng.integers(0, vocab, size=0 if empty else int(rng.integers(0, L + 1)))
                     for k, L in lens.items()}
        for k in lens:
            offs[k].append(pos[k])
            vals[k].append(state[k])
            pos[k] += state[k].size
    return ({k: np.concatenate(v).astype(np.int64) for k, v in vals.items()},
            {k: np.array(o, np.int64) for k, o in offs.items()})


def _oracle_out(vals, offs, keys, w, ws):
    per_key = [(w[k][vals[k]], offs[k]) for k in keys]
    out, _ = oracle.attention_pool(per_key, *ws)
    return out


@pytest.mark.parametrize("d", [64, 128])
def test_attention_pool_dedup_matches_oracle_and_kjt(d):
    rng = np.random.default_rng(d)
    b, vocab = 600, 3000
    keys = ["hist_a", "hist_b"]
    vals, offs = _grouped_batch(rng, b, vocab, {"hist_a": 32, "hist_b": 32})
    w = {k: rng.uniform(-0.1, 0.1, size=(vocab, d)).astype(np.float32) for k in keys}
    ws = [rng.standard_normal((d, d)).astype(np.float32) / np.sqrt(d) for _ in range(4)]
    tables = {k: R.EmbeddingTable(k, vocab, d, torch.as_tensor(w[k], device="cuda")) for k in keys}
    enc = R.DedupAttentionPool(tables, *ws)
    kjt = R.KJT(b, {k: R.JaggedTensor(vals[k], offs[k]) for k in keys})
    ik = R.kjt_to_ikjt(kjt, keys)
    got = enc(ik).cpu().numpy()
    base = enc(kjt).cpu().numpy()
    np.testing.assert_array_equal(got, base)          # dedup == baseline, bit for bit
    ref = _oracle_out(vals, offs, keys, w, ws)        # fp32 oracle over all B rows
    scale = float(np.abs(ref).max())
    np.testing.assert_allclose(got, ref, rtol=3e-2, atol=3e-2 * scale)
    # empty rows (both lists empty) are exactly zero
    empty = (np.diff(np.append(offs[keys[0]], vals[keys[0]].size)) == 0) & \
            (np.diff(np.append(offs[keys[1]], vals[keys[1]].size)) == 0)
    assert empty.any()
    assert not got[empty].any()


def test_attention_pool_long_rows_single_key():
    """n > 64 (several query/key blocks) and n > 1024 (key chunks)."""
    rng = np.random.default_rng(5)
    d, vocab = 128, 5000
    lens = [1, 63, 64, 65, 130, 700, 1100, 0, 17]
    vals = np.concatenate([rng.integers(0, vocab, size=n) for n in lens]).astype(np.int64)
    offs = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.int64)
    w = rng.uniform(-0.1, 0.1, size=(vocab, d)).astype(np.float32)
    ws = [rng.standard_normal((d, d)).astype(np.float32) / np.sqrt(d) for _ in range(4)]
    enc = R.DedupAttentionPool({"k": R.EmbeddingTable("k", vocab, d, torch.as_tensor(w, device="cuda"))},
                               *ws)
    got = enc(R.KJT(len(lens), {"k": R.JaggedTensor(vals, offs)})).cpu().numpy()
    ref, _ = oracle.attention_pool([(w[vals], offs)], *ws)
    scale = float(np.abs(ref).max())
    np.testing.assert_allclose(got, ref, rtol=3e-2, atol=3e-2 * scale)


def test_attention_pool_bad_id_message():
    d, vocab = 64, 100
    t = R.EmbeddingTable("k", vocab, d, torch.zeros((vocab, d), device="cuda"))
    ws = [np.eye(d, dtype=np.float32)] * 4
    enc = R.DedupAttentionPool({"k": t}, *ws)
    kjt = R.KJT(2, {"k": R.JaggedTensor(np.array([1, 2, 100], np.int64), np.array([0, 2], np.int64))})
    with pytest.raises(ValueError, match=r"feature 'k': ID 100 at position 2 out of range \[0, 100\)"):
        enc(kjt)
