"""Phase timeline of the cooperative GroupNorm (gn_fused) at the c2 shapes (needs the
ADX_GN_TIMELINE variant: tools/build_variant.sh gtl "-DADX_GN_TIMELINE" unet_kernels; run with
ADX_LIB_VARIANT=gtl).  Stamps: 0 start, 1 after griddepcontrol.wait, 2 chunk loaded + per-row
sums, 3 partials published, 4 after the grid barrier, 5 statistics folded, 6 applied + stored."""
import ctypes as C, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2406_06911_b200 as adx
from paper_2406_06911_b200 import _lib
P16, PF = C.POINTER(C.c_uint16), C.POINTER(C.c_float)
L = adx.lib()
for (HW, c0, c1) in ((9216, 320, 0), (9216, 320, 320), (2304, 640, 0), (576, 1280, 0), (144, 1280, 1280)):
    C_ = c0 + c1
    x0 = np.full((1, HW, c0), 0x3c00, np.uint16); x1 = np.full((1, HW, max(c1, 1)), 0x3c00, np.uint16)
    g = np.ones(C_, np.float32); b = np.zeros(C_, np.float32); o = np.zeros((1, HW, C_), np.uint16)
    ms = C.c_double()
    for _ in range(2):
        _lib.check(L.adx_group_norm_bf16(0, 1, HW, c0, c1, 32, x0.ctypes.data_as(P16),
                                         x1.ctypes.data_as(P16) if c1 else None, g.ctypes.data_as(PF),
                                         b.ctypes.data_as(PF), 1e-5, 1, o.ctypes.data_as(P16), 10, C.byref(ms)))
    buf = np.zeros((256, 8), np.uint64)
    _lib.check(L.adx_gn_timeline(buf.ctypes.data_as(C.POINTER(C.c_ulonglong)), 256))
    t = buf.astype(np.int64); t = t[t[:, 0] > 0]
    rel = (t - t[:, 0].min()) / 1e3
    med = np.median(rel, axis=0); mx = rel.max(axis=0)
    print(f"GN HW={HW} C={c0}+{c1}: {ms.value*1e3:.1f} us/launch (graph) | ctas {len(t)} | median "
          + " ".join(f"{x:.2f}" for x in med[:7]) + " | max " + " ".join(f"{x:.2f}" for x in mx[:7]), flush=True)
