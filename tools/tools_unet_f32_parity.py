"""ADX_F32 (and ADX_BF16) UNet modes vs the numpy oracle: per-step eps rel-L2 and the
final-latent rel-L2 of a full trajectory, at two sizes; plus the f32-mode pass time at c2."""
import json, sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2406_06911_b200 as adx
from oracle import oracle as O
from oracle.unet_oracle import UNetOracle

rel = lambda a, b: float(np.linalg.norm(a - b) / (np.linalg.norm(b) + 1e-30))
out = {}
for name, spec, T in (("small", dict(H=16, W=16, ch=(64, 128), attn=(1, 0), n_res=1, ctx_len=8, ctx_dim=64,
                                     temb_dim=128, seed=5), 4),
                      ("medium", dict(H=32, W=32, ch=(128, 256, 256), attn=(1, 1, 0), n_res=1, ctx_len=77,
                                      ctx_dim=256, temb_dim=256, seed=7), 6)):
    m = adx.build_unet_denoiser(**spec)
    s = adx.build_schedule(T, 0.01, 0.19)
    x = adx.Latent(O.random_normals(12, m.data_dim()).astype(np.float64), T)
    for prec, exact in (("f32", True), ("bf16", False)):
        traj = adx.sequential_denoise(m, x, s, precision=prec)
        orc = UNetOracle(spec, exact=exact)
        lat = x.values.astype(np.float64)
        eps_rel = []
        for k, t in enumerate(range(T, 0, -1)):
            eps = orc.eval_full(lat if exact else lat.astype(np.float32), t)
            eps_rel.append(rel(traj.eps_used[k], eps))
            lat = O.ddim_step(lat, np.asarray(eps, np.float64), t, s.alpha_bars)
        out[f"{name}_{prec}"] = {"T": T, "eps_rel_l2_max": max(eps_rel), "final_latent_rel_l2": rel(traj.latents[-1].values, lat),
                                 "oracle": "fp64" if exact else "fp32 with bf16 storage rounding"}
        print(name, prec, json.dumps(out[f"{name}_{prec}"]), flush=True)
m = adx.build_unet_denoiser(seed=0)
for prec in ("bf16", "f32"):
    ms, _, n = adx.time_model_pass(m, 50, 1, prec, [0])
    out[f"c2_pass_ms_{prec}"] = ms
    print("c2 pass", prec, ms, "ms", flush=True)
json.dump(out, open(sys.argv[1] if len(sys.argv) > 1 else "unet_parity.json", "w"), indent=1)
