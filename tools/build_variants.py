import os
import sys
from pathlib import Path

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_05239_b200.build import build  # noqa: E402

V = {
    "b6m4": ["RECD_SC_BATCH=6", "RECD_SCATTER_MINB=4"],
    "b5m4": ["RECD_SC_BATCH=5", "RECD_SCATTER_MINB=4"],
    "b7m4": ["RECD_SC_BATCH=7", "RECD_SCATTER_MINB=4"],
    "b6m4rs6": ["RECD_SC_BATCH=6", "RECD_SCATTER_MINB=4", "RECD_SC_RS=6"],
    "b6m4rs4": ["RECD_SC_BATCH=6", "RECD_SCATTER_MINB=4", "RECD_SC_RS=4"],
}
only = sys.argv[1:] or list(V)
for k in only:
    print(build(defines=V[k], out=Path(f"build/variants/librecd_{k}.so"), tag="_" + k))
