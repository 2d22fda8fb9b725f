"""(bn, split-K) sweep of the small-M launches of a c2 pass (12x12 level-3 / mid convs and the
M=144 GEMMs, 24x24 convs) -- where the tile plan leaves the most time on the table."""
import ctypes as C, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2406_06911_b200 as adx
from paper_2406_06911_b200 import _lib
P16 = C.POINTER(C.c_uint16)
L = adx.lib()
def conv(H, W, Ci, Co, bn, S):
    X = np.ones((1, H, W, Ci), np.uint16) * 0x3c00; Wt = np.ones((Co, 9 * Ci), np.uint16) * 0x3c00
    ms = C.c_double()
    _lib.check(L.adx_tc_plan_override(bn, S))
    _lib.check(L.adx_tc_conv3x3(0, 1, H, W, Ci, Co, X.ctypes.data_as(P16), Wt.ctypes.data_as(P16), None, None, 10, C.byref(ms)))
    return ms.value * 1e3
def gemm(M, N, K, bn, S):
    A = np.ones((M, K), np.uint16) * 0x3c00; B = np.ones((N, K), np.uint16) * 0x3c00
    ms = C.c_double()
    _lib.check(L.adx_tc_plan_override(bn, S))
    _lib.check(L.adx_tc_gemm(0, M, N, K, A.ctypes.data_as(P16), B.ctypes.data_as(P16), None, 0, None, 0, 10, C.byref(ms)))
    return ms.value * 1e3
for (H, W, Ci, Co) in ((12, 12, 1280, 1280), (24, 24, 1280, 1280)):
    res = {}
    for bn in (64, 128, 256):
        for S in (1, 2, 4, 8):
            try:
                res[(bn, S)] = round(conv(H, W, Ci, Co, bn, S), 1)
            except Exception as e:
                res[(bn, S)] = str(e)[:30]
    wb = Co * 9 * Ci * 2
    print("conv", H, W, Ci, Co, "weights MB", wb / 1e6, "floor us", round(wb / 6.5e6, 1), res, flush=True)
for (M, N, K) in ((144, 1280, 1280), (144, 10240 // 2, 1280), (576, 1280, 1280)):
    res = {}
    for bn in (64, 128, 256):
        for S in (1, 2, 4, 8):
            try:
                res[(bn, S)] = round(gemm(M, N, K, bn, S), 1)
            except Exception as e:
                res[(bn, S)] = str(e)[:30]
    print("gemm", M, N, K, res, flush=True)
_lib.check(L.adx_tc_plan_override(0, 0))
