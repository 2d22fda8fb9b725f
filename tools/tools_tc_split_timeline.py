import ctypes as C, sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2406_06911_b200 as adx
from paper_2406_06911_b200 import _lib
P16, PF = C.POINTER(C.c_uint16), C.POINTER(C.c_float)
L = adx.lib()
for (H, W, Ci, Co, bn, S) in ((12, 12, 1280, 1280, 128, 6), (48, 48, 640, 640, 160, 2), (24, 24, 1280, 1280, 160, 3)):
    X = np.ones((1, H, W, Ci), np.uint16) * 0x3c00; Wt = np.ones((Co, 9 * Ci), np.uint16) * 0x3c00
    R = np.ones((1, H, W, Co), np.uint16) * 0x3c00; O = np.zeros((1, H, W, Co), np.uint16)
    bias = np.zeros(Co, np.float32)
    for _ in range(2):
        _lib.check(L.adx_tc_conv3x3_bf16(0, 1, H, W, Ci, Co, X.ctypes.data_as(P16), Wt.ctypes.data_as(P16),
                                         bias.ctypes.data_as(PF), R.ctypes.data_as(P16), O.ctypes.data_as(P16), bn, S, 0, None))
    m_t = {12: 2, 48: 18, 24: 5}[H] if H != 48 else 18
    ctas = 300
    buf = np.zeros((ctas, 8), np.uint64)
    _lib.check(L.adx_tc_timeline(buf.ctypes.data_as(C.POINTER(C.c_ulonglong)), ctas))
    t = buf.astype(np.int64); used = t[:, 0] > 0; t = t[used]
    rel = (t - t[:, 0].min()) / 1e3
    med = np.median(rel, axis=0); mx = rel.max(axis=0)
    print(f"conv {H}x{W}x{Ci}->{Co} bn={bn} S={S} ctas={used.sum()}: median " + " ".join(f"{x:.2f}" for x in med) + " | max " + " ".join(f"{x:.2f}" for x in mx))
