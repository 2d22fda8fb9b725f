"""tcgen05 GEMM / conv3x3 throughput sweep (run on the GPU box)."""
import ctypes as C, json, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2406_06911_b200 as adx
from paper_2406_06911_b200 import _lib
P16 = C.POINTER(C.c_uint16); PF = C.POINTER(C.c_float)
rows = []
GEMMS = [(8192, 8192, 8192, 256)]
for L, Cc in ((9216, 320), (2304, 640), (576, 1280)):  # SD-2.1 transformer GEMMs per level
    GEMMS += [(L, Cc, Cc, 0), (L, 3 * Cc, Cc, 0), (L, 8 * Cc, Cc, 0), (L, Cc, 4 * Cc, 0)]
for (M, N, K, bn) in GEMMS:
    A = np.ones((M, K), np.uint16) * 0x3c00; B = np.ones((N, K), np.uint16) * 0x3c00
    ms = C.c_double()
    _lib.check(adx.lib().adx_tc_gemm(0, M, N, K, A.ctypes.data_as(P16), B.ctypes.data_as(P16), None, 0, None, bn, 10,
                                     C.byref(ms)))
    rows.append(dict(kind="gemm", M=M, N=N, K=K, bn=bn, us=round(ms.value * 1e3, 1), tflops=round(2 * M * N * K / ms.value / 1e9, 1)))
for (b, H, W, Ci, Co) in [(1, 96, 96, 320, 320), (1, 96, 96, 640, 320), (1, 48, 48, 640, 640), (1, 48, 48, 1280, 640),
                          (1, 24, 24, 1280, 1280), (1, 24, 24, 2560, 1280), (1, 12, 12, 1280, 1280),
                          (1, 12, 12, 2560, 1280)]:
    X = np.ones((b, H, W, Ci), np.uint16) * 0x3c00; Wt = np.ones((Co, 9 * Ci), np.uint16) * 0x3c00
    ms = C.c_double()
    _lib.check(adx.lib().adx_tc_conv3x3(0, b, H, W, Ci, Co, X.ctypes.data_as(P16), Wt.ctypes.data_as(P16), None, None, 10,
                                        C.byref(ms)))
    rows.append(dict(kind="conv3x3", b=b, H=H, W=W, Cin=Ci, Cout=Co, us=round(ms.value * 1e3, 1),
                     tflops=round(2 * b * H * W * Co * 9 * Ci / ms.value / 1e9, 1)))
for r in rows: print(json.dumps(r))
