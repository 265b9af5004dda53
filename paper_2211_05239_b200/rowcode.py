"""Row-delta coded host -> device copy of KJT batches (include/recd_host.h).

Session-clustered batches repeat or shift most history rows from one sample
to the next, and the end-to-end step is bound by the PCIe copy of the full
int64 KJT.  `encode` (librecd_host, C++ threads) turns each feature's rows
into one code per row plus the IDs the device cannot rebuild; librecd's
`recd_rowcode_decode` rebuilds the values on the device, exactly.
`staging.H2DPipeline(step, rowcode=True)` copies batches this way.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

__all__ = ["KEY", "REPEAT", "SHIFT", "load_host", "encode", "decode_reference"]

KEY, REPEAT, SHIFT = 0, 1, 2
_PATH = Path(os.environ.get("RECD_HOST_LIB", Path(__file__).resolve().parent / "librecd_host.so"))
_host = None


def load_host():
    global _host
    if _host is None:
        if not _PATH.exists():
            raise ImportError(f"{_PATH} is missing: run paper_2211_05239_b200.build")
        lib = C.CDLL(str(_PATH))
        pp = C.POINTER(C.c_void_p)
        lib.recd_rowcode_encode.restype = C.c_int32
        lib.recd_rowcode_encode.argtypes = [C.c_int32, C.c_int64, pp, pp, C.POINTER(C.c_int64), pp,
                                            pp, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                            C.c_int32]
        _host = lib
    return _host


def _ptr(x) -> int:
    return x.data_ptr() if hasattr(x, "data_ptr") else x.ctypes.data


def encode(values, offsets, batch_size: int, codes_out, lits_out, num_threads: int = 0):
    """values/offsets: per feature int64 host arrays (numpy or CPU tensors);
    codes_out: per feature uint8[batch_size]; lits_out: per feature int64
    buffers.  Returns the literal count of every feature."""
    F = len(values)
    lib = load_host()
    if num_threads <= 0:
        num_threads = int(os.environ.get("RECD_ROWCODE_THREADS", "0"))
    arr = lambda xs: (C.c_void_p * F)(*[_ptr(x) for x in xs])  # noqa: E731
    nv = (C.c_int64 * F)(*[int(v.shape[0]) for v in values])
    caps = (C.c_int64 * F)(*[int(x.shape[0]) for x in lits_out])
    cnt = (C.c_int64 * F)()
    rc = lib.recd_rowcode_encode(F, int(batch_size), arr(values), arr(offsets), nv, arr(codes_out),
                                 arr(lits_out), caps, cnt, int(num_threads))
    if rc == 2:
        raise ValueError("row-coded literals exceed the buffer capacity")
    if rc != 0:
        raise ValueError("recd_rowcode_encode: invalid arguments")
    return list(cnt)


def decode_reference(codes: np.ndarray, offsets: np.ndarray, n_values: int,
                     lits: np.ndarray) -> np.ndarray:
    """Host restatement of the device decode (for tests): row r is
    lits[c(r) - L_r : c(r)] with c the inclusive prefix of literal counts."""
    lens = np.diff(np.append(offsets, n_values))
    cnt = np.where(codes == KEY, lens, np.where(codes == SHIFT, 1, 0))
    base = np.cumsum(cnt) - lens
    out = np.empty(n_values, dtype=np.int64)
    for r in range(len(offsets)):
        out[offsets[r]: offsets[r] + lens[r]] = lits[base[r]: base[r] + lens[r]]
    return out
