import os
import sys
from pathlib import Path

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_05239_b200.build import build  # noqa: E402

V = {
    "memset": ["RECD_OS_SETUP_CLEAR=0"],
    "cpilp8": ["RECD_CP_ILP=8"],
    "gu256": ["RECD_GU_CH=256"],
    "os12": ["RECD_OS_ITEMS=12"],
    "noil": ["RECD_OS_IL=0"],
    "lb16": ["RECD_OS_LB=16"],
    "lb4": ["RECD_OS_LB=4"],
    "noearly": ["RECD_OS_EARLY=0"],
    "notiny": ["RECD_TINY_CH=0"],
    "rs256": ["RECD_RS_SMALLB=0"],
    "gu16": ["RECD_GU_CH_SMALL=16"],
    "gu16rc32": ["RECD_GU_CH_SMALL=16", "RECD_RC_SMALL=32"],
    "nbbig": ["RECD_NB_SMALL=0"],
    "nolocal": ["RECD_OS_LOCAL=0"],
    "rc32": ["RECD_RC_SMALL=32"],
    "nocoal": ["RECD_RS_COAL=0"],
    "noflat": ["RECD_GU_FLAT=0"],
    "fm4": ["RECD_GUF_MINB=4"],
    "rs8": ["RECD_SC_RS=8"],
    "rs4": ["RECD_SC_RS=4"],
    "noxcs": ["RECD_EXPAND_CS=0"],
    "gcs": ["RECD_GUF_CS=1"],
    "xrf16": ["RECD_EXPAND_RF=16"],
    "xrf4": ["RECD_EXPAND_RF=4"],
    "sp4m4": ["RECD_SC_PIPE=1", "RECD_SC_BATCH=4", "RECD_SCATTER_MINB=4"],
    "sp4m3": ["RECD_SC_PIPE=1", "RECD_SC_BATCH=4", "RECD_SCATTER_MINB=3"],
    "sp6m3": ["RECD_SC_PIPE=1", "RECD_SC_BATCH=6", "RECD_SCATTER_MINB=3"],
    "sp3m4": ["RECD_SC_PIPE=1", "RECD_SC_BATCH=3", "RECD_SCATTER_MINB=4"],
    "screv": ["RECD_SC_REV=1"],
    "rsold": ["RECD_RS_SHORT=0"],
    "os12m4": ["RECD_OS_ITEMS=12", "RECD_OS_MINB=4"],
    "os8m5": ["RECD_OS_ITEMS=8", "RECD_OS_MINB=5"],
    "os16m4": ["RECD_OS_MINB=4"],
    "oslb16": ["RECD_OS_LB=16"],
    "notma": ["RECD_RS_TMA=0"],
    "rsm5": ["RECD_RS_MINB=5"],
    "nohist": ["RECD_OCC_HIST=0"],
    "sl1": ["RECD_SCATTER_L2=1"],
    "sl0": ["RECD_SCATTER_L2=0"],
    "rsm6": ["RECD_RS_MINB=6"],
    "ca2": ["RECD_RING_CA=1"],
    "ca1m3": ["RECD_RING_CA=1", "RECD_RING_K=1"],
    "ca1m4": ["RECD_RING_CA=1", "RECD_RING_K=1", "RECD_RING_MINB=4"],
    "k1m4": ["RECD_RING_K=1", "RECD_RING_MINB=4"],
    "cp32": ["RECD_CP_IT=32", "RECD_OC_CH=8192"],
    "cp64": ["RECD_CP_IT=64", "RECD_OC_CH=16384"],
    "b8m3": ["RECD_SC_BATCH=8", "RECD_SCATTER_MINB=3"],
    "b8r4": ["RECD_SC_BATCH=8", "RECD_SC_RS=4"],
    "b4": ["RECD_SC_BATCH=4"],
    "r4": ["RECD_SC_RS=4"],
    "r8": ["RECD_SC_RS=8"],
    "b10m3": ["RECD_SC_BATCH=10", "RECD_SCATTER_MINB=3"],
}
only = sys.argv[1:] or list(V)
for k in only:
    print(build(defines=V[k], out=Path(f"build/variants/librecd_{k}.so"), tag="_" + k))
