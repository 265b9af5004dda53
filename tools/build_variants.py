import os
import sys
from pathlib import Path

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_05239_b200.build import build  # noqa: E402

V = {
    "noring": ["RECD_POOL_RING=0"],
    "nb1m3": ["RECD_RING_K=1", "RECD_RING_MINB=3"],
    "nb3m2": ["RECD_RING_K=3", "RECD_RING_MINB=2"],
    "nb4m1": ["RECD_RING_K=4", "RECD_RING_MINB=1"],
}
only = sys.argv[1:] or list(V)
for k in only:
    print(build(defines=V[k], out=Path(f"build/variants/librecd_{k}.so"), tag="_" + k))
