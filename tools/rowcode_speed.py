import sys, time, numpy as np
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import bench
from paper_2211_05239_b200 import rowcode
args = bench.parse([])
batch = bench.make_batch(args, 0, 1)
keys = list(batch.keys)
B = args.batch
vals = [batch.values[k] for k in keys]; offs = [batch.offsets[k] for k in keys]
codes = [np.empty(B, np.uint8) for _ in keys]
lits = [np.empty(v.size, np.int64) for v in vals]
for th in (1, 4, 8, 16, 0):
    ts = []
    for _ in range(5):
        t0 = time.perf_counter(); cnt = rowcode.encode(vals, offs, B, codes, lits, th); ts.append(time.perf_counter() - t0)
    print("threads", th, "ms", round(min(ts)*1e3, 2), "lits", sum(cnt), "of", sum(v.size for v in vals))
# check exactness on a few features
for f in (0, 5, 25):
    dec = rowcode.decode_reference(codes[f], offs[f], vals[f].size, lits[f])
    assert np.array_equal(dec, vals[f]), f
print("ok")
