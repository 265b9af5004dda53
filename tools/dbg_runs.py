import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2211_05239_b200 as R
rng = np.random.default_rng(1)
b, rows, dim = 2000, 500, 1
vals, offs, pos, state = [], [], 0, None
for i in range(b):
    if state is None or rng.random() > 0.8:
        state = rng.integers(0, rows, size=int(rng.integers(0, 13)))
    offs.append(pos); vals.append(state); pos += state.size
v = np.concatenate(vals).astype(np.int64); o = np.array(offs, np.int64)
ik = R.kjt_to_ikjt(R.KJT(b, {"k": R.JaggedTensor(v, o)}), ["k"])
w = rng.uniform(-0.1, 0.1, size=(rows, dim)).astype(np.float32)
t = R.EmbeddingTable("k", rows, dim, torch.as_tensor(w, device="cuda"))
g = torch.randn(b, dim, device="cuda")
[(ids, grads)] = R.pooled_lookup_backward([ik.per_feature["k"]], [t], "sum", [g], inverses=[ik.inverse_lookup])
torch.cuda.synchronize()
print("ids", ids.numel(), ids[:10].tolist())
