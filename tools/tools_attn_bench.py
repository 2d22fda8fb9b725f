"""Fused attention alone at the UNet self-attention shapes (graph-timed, 10 launches);
ADX_ATTN_SPLITS=S forces the split-KV factor."""
import ctypes as C, numpy as np, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_06911_b200 as adx
from paper_2406_06911_b200 import _lib
P16 = C.POINTER(C.c_uint16)
shapes = ((9216, 9216, 320), (2304, 2304, 640), (576, 576, 1280), (9216, 77, 320), (2304, 77, 640), (576, 77, 1280))
for L, Lk, C_ in shapes:
    q = np.ones((max(L, Lk), C_), np.uint16) * 0x3c00; v = np.ones((Lk, C_), np.uint16) * 0x3c00
    out = np.zeros((L, C_), np.uint16)
    ms = C.c_double()
    _lib.check(adx.lib().adx_tc_attention(0, L, Lk, C_, q.ctypes.data_as(P16), q.ctypes.data_as(P16),
                                          v.ctypes.data_as(P16), C_, out.ctypes.data_as(P16), 10, C.byref(ms)))
    print(L, Lk, C_, os.environ.get("ADX_ATTN_SPLITS", "auto"), round(ms.value * 1e3, 1), "us",
          round(4 * L * Lk * C_ / ms.value / 1e9, 1), "TFLOP/s")
