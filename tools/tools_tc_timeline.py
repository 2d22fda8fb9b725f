"""Per-CTA phase timeline of single tc_gemm / conv launches (needs the ADX_TC_TIMELINE variant:
tools/build_variant.sh tl "-DADX_TC_TIMELINE" tc_gemm; run with ADX_LIB_VARIANT=tl).
Stamps: 0 start, 1 prologue done, 2 after griddepcontrol.wait, 3 first k-block landed (MMA
warp), 4 accumulator ready (epilogue), 5 epilogue stores issued, 6 stores complete, 7 exit.
The launches use the UNet pass's epilogue: bf16 output (TMA-store staging where eligible) with
a bf16 residual.  The first launch of each shape is cold; the second one is shown."""
import ctypes as C, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2406_06911_b200 as adx
from paper_2406_06911_b200 import _lib
P16, PF = C.POINTER(C.c_uint16), C.POINTER(C.c_float)
L = adx.lib()
def show(name, ctas):
    buf = np.zeros((ctas, 8), np.uint64)
    _lib.check(L.adx_tc_timeline(buf.ctypes.data_as(C.POINTER(C.c_ulonglong)), ctas))
    t = buf.astype(np.int64)
    rel = (t - t[:, 0].min()) / 1e3  # us
    med = np.median(rel, axis=0)
    print(f"{name}: ctas={ctas} median stamps (us): " + " ".join(f"{x:.2f}" for x in med)
          + f" | mainloop {med[4]-med[3]:.2f} epilogue {med[5]-med[4]:.2f} | last exit {rel[:, 7].max():.2f}", flush=True)
for (M, N, K, bn, ctas) in ((144, 1280, 1280, 64, 40), (576, 1280, 1280, 64, 100), (9216, 320, 320, 160, 144),
                            (2304, 640, 640, 80, 144)):
    A = np.ones((M, K), np.uint16) * 0x3c00; B = np.ones((N, K), np.uint16) * 0x3c00
    R = np.ones((M, N), np.uint16) * 0x3c00; O = np.zeros((M, N), np.uint16); bias = np.zeros(N, np.float32)
    for _ in range(2):
        _lib.check(L.adx_tc_gemm_bf16(0, M, N, K, A.ctypes.data_as(P16), B.ctypes.data_as(P16), bias.ctypes.data_as(PF),
                                      R.ctypes.data_as(P16), N, O.ctypes.data_as(P16), N, bn, 1, 0, None))
    show(f"gemm {M}x{N}x{K} bn={bn} (+res, bf16)", ctas)
for (H, W, Ci, Co, ctas) in ((96, 96, 320, 320, 144), (48, 48, 640, 640, 144), (12, 12, 1280, 1280, 80)):
    X = np.ones((1, H, W, Ci), np.uint16) * 0x3c00; Wt = np.ones((Co, 9 * Ci), np.uint16) * 0x3c00
    R = np.ones((1, H, W, Co), np.uint16) * 0x3c00; O = np.zeros((1, H, W, Co), np.uint16)
    bias = np.zeros(Co, np.float32)
    for _ in range(2):
        _lib.check(L.adx_tc_conv3x3_bf16(0, 1, H, W, Ci, Co, X.ctypes.data_as(P16), Wt.ctypes.data_as(P16),
                                         bias.ctypes.data_as(PF), R.ctypes.data_as(P16), O.ctypes.data_as(P16), 0, 0, 0, None))
    show(f"conv {H}x{W}x{Ci}->{Co} (+res, bf16)", ctas)
