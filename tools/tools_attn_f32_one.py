"""One level-0 self-attention in the f32 parity mode (split-operand kernel, L=9216, C=320) for ncu."""
import ctypes as C, numpy as np, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_06911_b200 as adx
from paper_2406_06911_b200 import _lib
PF = C.POINTER(C.c_float)
rng = np.random.default_rng(0)
L, Cc = 9216, 320
q = rng.standard_normal((L, Cc)).astype(np.float32); o = np.zeros((L, Cc), np.float32)
_lib.check(adx.lib().adx_tc_attention_f32(0, 1, L, L, Cc, q.ctypes.data_as(PF), q.ctypes.data_as(PF),
                                          q.ctypes.data_as(PF), o.ctypes.data_as(PF), 0, None))
print("ok")
