"""One level-0 conv3x3 (96x96, 320->320) and one level-0 self-attention (L=9216, C=320) for ncu --set full."""
import ctypes as C, numpy as np, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_06911_b200 as adx
from paper_2406_06911_b200 import _lib
P16 = C.POINTER(C.c_uint16); PF = C.POINTER(C.c_float)
rng = np.random.default_rng(0)
bf = lambda a: (np.ascontiguousarray(a, np.float32).view(np.uint32) >> 16).astype(np.uint16)
X = bf(rng.standard_normal((1, 96, 96, 320))); Wt = bf(rng.standard_normal((320, 9 * 320)) / 54.0)
out = np.zeros((1, 96, 96, 320), np.float32)
_lib.check(adx.lib().adx_tc_conv3x3(0, 1, 96, 96, 320, 320, X.ctypes.data_as(P16), Wt.ctypes.data_as(P16), None,
                                    out.ctypes.data_as(PF), 0, None))
L, Cc = 9216, 320
q = bf(rng.standard_normal((L, Cc))); vt = bf(rng.standard_normal((Cc, L))); o = np.zeros((L, Cc), np.uint16)
_lib.check(adx.lib().adx_tc_attention(0, L, L, Cc, q.ctypes.data_as(P16), q.ctypes.data_as(P16), vt.ctypes.data_as(P16),
                                      Cc, o.ctypes.data_as(P16), 0, None))
print("ok")
