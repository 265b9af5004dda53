import os
import sys
from pathlib import Path

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_05239_b200.build import build  # noqa: E402

V = {
    "scb4": ["RECD_SCATTER_MINB=4"],
    "scrs4": ["RECD_SC_RS=4"],
    "rk3": ["RECD_RING_K=3", "RECD_RING_MINB=2"],
    "rk1": ["RECD_RING_K=1", "RECD_RING_MINB=4"],
    "osb4": ["RECD_OS_MINB=4"],
}
only = sys.argv[1:] or list(V)
for k in only:
    print(build(defines=V[k], out=Path(f"build/variants/librecd_{k}.so"), tag="_" + k))
