import os
import sys
from pathlib import Path

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_05239_b200.build import build  # noqa: E402

V = {
    "a": ["RECD_POOL_VW=2", "RECD_POOL_MINB=3", "RECD_BWD_VW=2", "RECD_SCATTER_MINB=3"],
    "b": ["RECD_POOL_VW=4", "RECD_POOL_MINB=2", "RECD_BWD_VW=4", "RECD_SCATTER_MINB=3"],
    "c": ["RECD_POOL_VW=4", "RECD_POOL_MINB=2", "RECD_BWD_VW=4", "RECD_SCATTER_MINB=2"],
    "d": ["RECD_POOL_VW=2", "RECD_POOL_MINB=2", "RECD_BWD_VW=2", "RECD_SCATTER_MINB=2"],
}
only = sys.argv[1:] or list(V)
for k in only:
    print(build(defines=V[k], out=Path(f"build/variants/librecd_{k}.so"), tag="_" + k))
