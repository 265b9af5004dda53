import os
import sys
from pathlib import Path

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_05239_b200.build import build  # noqa: E402

V = {
    "s2m2": ["RECD_POOL_STREAM=1", "RECD_STREAM_G=2", "RECD_STREAM_MINB=2"],
    "s3m2": ["RECD_POOL_STREAM=1", "RECD_STREAM_G=3", "RECD_STREAM_MINB=2"],
    "s4m1": ["RECD_POOL_STREAM=1", "RECD_STREAM_G=4", "RECD_STREAM_MINB=1"],
    "s2m3v2": ["RECD_POOL_STREAM=1", "RECD_STREAM_G=2", "RECD_STREAM_MINB=3", "RECD_POOL_VW=2"],
}
only = sys.argv[1:] or list(V)
for k in only:
    print(build(defines=V[k], out=Path(f"build/variants/librecd_{k}.so"), tag="_" + k))
