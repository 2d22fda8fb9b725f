import ctypes as C, numpy as np, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_06911_b200 as adx
from paper_2406_06911_b200 import _lib
P16 = C.POINTER(C.c_uint16)
for L, C_ in ((9216, 320), (2304, 640), (576, 1280)):
    q = np.ones((L, C_), np.uint16) * 0x3c00; vt = np.ones((C_, L), np.uint16) * 0x3c00; out = np.zeros((L, C_), np.uint16)
    ms = C.c_double()
    _lib.check(adx.lib().adx_tc_attention(0, L, L, C_, q.ctypes.data_as(P16), q.ctypes.data_as(P16), vt.ctypes.data_as(P16), C_, out.ctypes.data_as(P16), 10, C.byref(ms)))
    print(L, C_, round(ms.value*1e3,1), "us", round(4*L*L*C_/ms.value/1e9,1), "TFLOP/s")
