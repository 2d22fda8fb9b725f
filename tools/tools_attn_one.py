"""One fused-attention launch (L=9216, C=320) for ncu."""
import ctypes as C, numpy as np, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_06911_b200 as adx
from paper_2406_06911_b200 import _lib
P16 = C.POINTER(C.c_uint16)
L, C_ = int(sys.argv[1]) if len(sys.argv) > 1 else 9216, 320
rng = np.random.default_rng(0)
q = (rng.standard_normal((L, C_)).astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)
vt = (rng.standard_normal((C_, L)).astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)
out = np.zeros((L, C_), np.uint16)
_lib.check(adx.lib().adx_tc_attention(0, L, L, C_, q.ctypes.data_as(P16), q.ctypes.data_as(P16), vt.ctypes.data_as(P16), C_, out.ctypes.data_as(P16), 0, None))
print("ok")
