"""Tile plans (N tile, split-K) for the stride-2 downsample convs of the headline config: graph-timed
sweep through adx_tc_conv3x3_s2_bf16; prints tc_plan_table.inc rows keyed {2, H_in, W_in, Cin, Cout}."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2406_06911_b200 as adx
L = adx.lib()
P16, PF = C.POINTER(C.c_uint16), C.POINTER(C.c_float)
for (H, W, Ci, Co) in [(96, 96, 320, 320), (48, 48, 640, 640), (24, 24, 1280, 1280)]:
    X = np.full((H, W, Ci), 0x3c00, np.uint16); Wt = np.full((Co, 9 * Ci), 0x3c00, np.uint16)
    b = np.zeros(Co, np.float32); O = np.zeros((H // 2, W // 2, Co), np.uint16)
    res = {}
    for bn in (0, 64, 80, 96, 128, 160, 192, 256):
        for s in ((0,) if bn == 0 else range(1, 9)):
            ms = C.c_double()
            rc = L.adx_tc_conv3x3_s2_bf16(0, 1, H, W, Ci, Co, X.ctypes.data_as(P16), Wt.ctypes.data_as(P16),
                                         b.ctypes.data_as(PF), O.ctypes.data_as(P16), bn, s, 20, C.byref(ms))
            if rc == 0:
                res[(bn, s)] = ms.value * 1e3
    best = min((v, k) for k, v in res.items() if k[0])
    print(f"    {{2, {H}, {W}, {Ci}, {Co}, {best[1][0]}, {best[1][1]}}},  // {best[0]:.1f} (model plan {res[(0, 0)]:.1f})",
          flush=True)
