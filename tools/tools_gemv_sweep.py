"""GEMV tuning sweep (run on the GPU box): ms/GEMV and GB/s per config."""
import ctypes as C, json, os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 1 and sys.argv[1] == "child":
    import paper_2406_06911_b200 as adx
    L = adx.lib()
    out = []
    for prec, wb in ((1, 4), (2, 2), (0, 8)):
        for n, chain in ((4096, 8), (8192, 4), (1024, 64), (256, 64)):
            for pdl in (1, 0):
                ms = C.c_double()
                adx._lib.check(L.adx_bench_gemv(0, prec, n, chain, 20, pdl, C.byref(ms)))
                gbs = n * ((n + 7) // 8 * 8) * wb / (ms.value * 1e-3) / 1e9
                out.append(dict(cfg=os.environ.get("ADX_GEMV_CFG", os.environ.get("ADX_GEMV", "0")), prec=prec, n=n,
                                pdl=pdl, us=round(ms.value * 1e3, 2), gbs=round(gbs)))
    print(json.dumps(out))
else:
    for env in ({"ADX_GEMV": "ldg"}, *({"ADX_GEMV_CFG": str(i)} for i in range(6))):
        e = dict(os.environ, **env)
        r = subprocess.run([sys.executable, __file__, "child"], env=e, capture_output=True, text=True)
        print(r.stdout.strip() or r.stderr[-2000:], flush=True)
