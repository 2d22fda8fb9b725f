"""Stream-K attention phase timeline (needs the -DADX_SK_TIMELINE variant: tools/build_variant.sh sktl
"-DADX_SK_TIMELINE" tc_attn; run with ADX_LIB_VARIANT=sktl).  Stamps of the first softmax thread per
CTA: 0 start; per segment q: 1+3q first S ready, 2+3q last block done, 3+3q output / record / combine done."""
import ctypes as C, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2406_06911_b200 as adx
from paper_2406_06911_b200 import _lib
P16 = C.POINTER(C.c_uint16)
L_ = adx.lib()
for (L, C_) in ((9216, 320), (2304, 640)):
    q = np.full((L, C_), 0x3c00, np.uint16); o = np.zeros((L, C_), np.uint16)
    for _ in range(2):
        _lib.check(L_.adx_tc_attention(0, L, L, C_, q.ctypes.data_as(P16), q.ctypes.data_as(P16), q.ctypes.data_as(P16),
                                       C_, o.ctypes.data_as(P16), 0, None))
    G = 296
    buf = np.zeros((G, 16), np.uint64)
    _lib.check(L_.adx_sk_timeline(buf.ctypes.data_as(C.POINTER(C.c_ulonglong)), G))
    t = buf.astype(np.int64)
    t0 = t[:, 0].min()
    rel = np.where(t > 0, (t - t0) / 1e3, np.nan)
    print(f"L={L} C={C_}: kernel span {np.nanmax(rel):.1f} us; start spread {np.nanmax(rel[:, 0]):.1f} us")
    for qq in range(4):
        a, b, c = rel[:, 1 + 3 * qq], rel[:, 2 + 3 * qq], rel[:, 3 + 3 * qq]
        if np.all(np.isnan(a)):
            break
        print(f"  segment {qq}: first S ready (med) {np.nanmedian(a):7.2f}  loop {np.nanmedian(b - a):7.2f}  "
              f"epilogue {np.nanmedian(c - b):6.2f} (max {np.nanmax(c - b):6.2f})  end (max) {np.nanmax(c):7.2f}  "
              f"ctas {np.sum(~np.isnan(a))}")
