import os
import sys
from pathlib import Path

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_05239_b200.build import build  # noqa: E402

V = {
    "ct16": ["RECD_SORT_CHUNK_TILES=16"],
    "ct32": ["RECD_SORT_CHUNK_TILES=32"],
    "it16ct4": ["RECD_SORT_ITEMS=16", "RECD_SORT_CHUNK_TILES=4"],
    "it16ct8": ["RECD_SORT_ITEMS=16", "RECD_SORT_CHUNK_TILES=8"],
    "it12ct8": ["RECD_SORT_ITEMS=12", "RECD_SORT_CHUNK_TILES=8"],
}
only = sys.argv[1:] or list(V)
for k in only:
    print(build(defines=V[k], out=Path(f"build/variants/librecd_{k}.so"), tag="_" + k))
