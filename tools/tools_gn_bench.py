"""GroupNorm(+SiLU) launch time at the UNet shapes (graph of 10 launches): the cluster kernel
(default) vs the previous path (ADX_GN_CLUSTER=0: cooperative one-launch for one image, stats +
apply for batches) -- run once per setting (the switch is read once per process)."""
import ctypes as C, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2406_06911_b200 as adx
from paper_2406_06911_b200 import _lib
P16, PF = C.POINTER(C.c_uint16), C.POINTER(C.c_float)
L = adx.lib()
for (B, HW, c0, c1) in ((1, 9216, 320, 0), (1, 9216, 320, 320), (1, 9216, 640, 320), (1, 2304, 640, 0),
                        (1, 2304, 640, 640), (1, 576, 1280, 0), (1, 576, 1280, 1280), (1, 144, 1280, 1280),
                        (2, 16384, 320, 0), (16, 4096, 320, 0)):
    C_ = c0 + c1
    x0 = np.full((B, HW, c0), 0x3c00, np.uint16); x1 = np.full((B, HW, max(c1, 1)), 0x3c00, np.uint16)
    g = np.ones(C_, np.float32); b = np.zeros(C_, np.float32); o = np.zeros((B, HW, C_), np.uint16)
    ms = C.c_double()
    _lib.check(L.adx_group_norm_bf16(0, B, HW, c0, c1, 32, x0.ctypes.data_as(P16), x1.ctypes.data_as(P16) if c1 else None,
                                     g.ctypes.data_as(PF), b.ctypes.data_as(PF), 1e-5, 1, o.ctypes.data_as(P16), 20,
                                     C.byref(ms)))
    mb = B * HW * C_ * 2 * 2 / 1e6
    print(f"GN cluster={os.environ.get('ADX_GN_CLUSTER', '1')} B={B} HW={HW} C={c0}+{c1}: {ms.value*1e3:.1f} us, "
          f"{mb / ms.value:.0f} GB/s (read + write)", flush=True)
