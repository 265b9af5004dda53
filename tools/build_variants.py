import os
import sys
from pathlib import Path

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_05239_b200.build import build  # noqa: E402

V = {
    "m4": ["RECD_OS_MINB=4"],
    "m2": ["RECD_OS_MINB=2"],
    "i12m4": ["RECD_OS_ITEMS=12", "RECD_OS_MINB=4"],
    "i8m5": ["RECD_OS_ITEMS=8", "RECD_OS_MINB=5"],
}
only = sys.argv[1:] or list(V)
for k in only:
    print(build(defines=V[k], out=Path(f"build/variants/librecd_{k}.so"), tag="_" + k))
