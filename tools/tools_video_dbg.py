import sys, time, numpy as np
sys.path.insert(0, "/root/repo")
import paper_2406_06911_b200 as adx
from oracle import oracle as O
def rel(a, b): return float(np.linalg.norm(a - b) / (np.linalg.norm(b) + 1e-12))
variants = [
    ("c5", dict(H=64, W=64, ctx_dim=768, frames=16, motion=True)),
    ("c5-nomotion", dict(H=64, W=64, ctx_dim=768, frames=16, motion=False)),
    ("c5-f4", dict(H=64, W=64, ctx_dim=768, frames=4, motion=True)),
    ("c5-f2", dict(H=64, W=64, ctx_dim=768, frames=2, motion=True)),
    ("32px-f16", dict(H=32, W=32, ctx_dim=768, frames=16, motion=True)),
    ("sd15-1", dict(H=64, W=64, ctx_dim=768)),
]
only = sys.argv[1:] 
for name, kw in variants:
    if only and name not in only: continue
    m = adx.build_unet_denoiser(seed=0, **kw)
    s = adx.build_schedule(2, 0.01, 0.19)
    x = adx.Latent(O.random_normals(12, m.data_dim()).astype(np.float64), 2)
    out = {}
    for prec in ("bf16", "f32"):
        try:
            tr = adx.sequential_denoise(m, x, s, precision=prec)
            e = tr.eps_used[0]
            out[prec] = e
            print(name, prec, "finite", bool(np.all(np.isfinite(e))), "norm", float(np.linalg.norm(e)), flush=True)
        except Exception as ex:
            print(name, prec, "ERR", ex, flush=True)
    if len(out) == 2:
        print(name, "rel bf16 vs f32", rel(out["bf16"], out["f32"]), flush=True)
    del m
