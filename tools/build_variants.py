import os
import sys
from pathlib import Path

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_05239_b200.build import build  # noqa: E402

V = {
    "nopref": ["RECD_RING_PREF=0"],
    "pref2": ["RECD_RING_PREF=2"],
    "k3": ["RECD_RING_PREF=0", "RECD_RING_K=3", "RECD_RING_MINB=2"],
}
only = sys.argv[1:] or list(V)
for k in only:
    print(build(defines=V[k], out=Path(f"build/variants/librecd_{k}.so"), tag="_" + k))
