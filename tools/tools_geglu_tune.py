"""Split-K plans for the fused-GEGLU GEMMs (ff1; the N tile is fixed at 2 x adx_tc_geglu_group()):
graph-timed sweep of S = 1..8 through adx_tc_gemm (act 2) under adx_tc_plan_override; prints
tc_plan_table.inc rows keyed {3, M, N, K, 0, bn, S}."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2406_06911_b200 as adx
L = adx.lib()
P16, PF = C.POINTER(C.c_uint16), C.POINTER(C.c_float)
bn = 2 * L.adx_tc_geglu_group()
shapes = [(144, 10240, 1280), (576, 10240, 1280), (2304, 5120, 640), (9216, 2560, 320),   # c2
          (2048, 10240, 1280), (8192, 5120, 640),                                        # c4
          (1024, 10240, 1280), (4096, 10240, 1280), (16384, 5120, 640), (65536, 2560, 320)]  # c5
for (M, N, K) in shapes:
    A = np.full((M, K), 0x3c00, np.uint16); B = np.full((N, K), 0x3c00, np.uint16)
    bias = np.zeros(N, np.float32); out = np.zeros((M, N // 2), np.float32)
    res = {}
    for s in range(0, 9):
        if s and (K // 64) // s < 1:
            continue
        L.adx_tc_plan_override(0, 0)
        if s:
            L.adx_tc_plan_override(bn, s)
        ms = C.c_double()
        rc = L.adx_tc_gemm(0, M, N, K, A.ctypes.data_as(P16), B.ctypes.data_as(P16), bias.ctypes.data_as(PF), 2,
                           out.ctypes.data_as(PF), 0, 20, C.byref(ms))
        L.adx_tc_plan_override(0, 0)
        if rc == 0:
            res[s] = ms.value * 1e3
    best = min((v, k) for k, v in res.items() if k)
    print(f"    {{3, {M}, {N}, {K}, 0, {bn}, {best[1]}}},  // {best[0]:.1f} (GEGLU, fp32 out; model plan {res[0]:.1f})",
          flush=True)
