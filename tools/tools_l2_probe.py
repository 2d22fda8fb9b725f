"""Is the tcgen05 conv mainloop L2-bandwidth-bound?  The 96x96x320->320 conv (144 tiles) with the
persistent grid capped at 144 / 72 / 36 CTAs (ADX_TC_MAXCTAS, set per process): per-k-block time
of the first tile from the timeline stamps (ADX_TC_TIMELINE variant)."""
import ctypes as C, os, subprocess, sys
code = r'''
import ctypes as C, sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2406_06911_b200 as adx
from paper_2406_06911_b200 import _lib
P16, PF = C.POINTER(C.c_uint16), C.POINTER(C.c_float)
L = adx.lib()
H, W, Ci, Co = 96, 96, 320, 320
BN = int(os.environ.get("BN", "160"))
X = np.ones((1, H, W, Ci), np.uint16) * 0x3c00; Wt = np.ones((Co, 9 * Ci), np.uint16) * 0x3c00
O = np.zeros((1, H, W, Co), np.uint16); bias = np.zeros(Co, np.float32)
ms = C.c_double()
for _ in range(2):
    _lib.check(L.adx_tc_conv3x3_bf16(0, 1, H, W, Ci, Co, X.ctypes.data_as(P16), Wt.ctypes.data_as(P16),
                                     bias.ctypes.data_as(PF), None, O.ctypes.data_as(P16), BN, 1, 5, C.byref(ms)))
n = int(os.environ.get("ADX_TC_MAXCTAS", "144"))
buf = np.zeros((n, 8), np.uint64)
_lib.check(L.adx_tc_timeline(buf.ctypes.data_as(C.POINTER(C.c_ulonglong)), n))
t = buf.astype(np.int64); rel = (t - t[:, 0].min()) / 1e3; med = np.median(rel, axis=0)
print(f"bn={BN} ctas={n}: launch {ms.value*1e3:.1f} us, first-tile mainloop {med[4]-med[3]:.2f} us = {1e3*(med[4]-med[3])/45:.0f} ns per k-block")
'''
for bn, n in ((160, 144), (160, 36), (64, 36), (128, 36), (256, 36)):
    env = dict(os.environ, ADX_TC_MAXCTAS=str(n), ADX_LIB_VARIANT="tl", BN=str(bn))
    print(subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True).stdout.strip(), flush=True)
