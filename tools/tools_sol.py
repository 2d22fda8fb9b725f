"""Per-launch speed-of-light table of one UNet pass (bench.roofline's per_launch_sol), plus the
slowest launches against their SOL.  usage: tools_sol.py [config, default c2] [precision, default bf16]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2406_06911_b200 as adx
import bench
cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
prec = sys.argv[2] if len(sys.argv) > 2 else "bf16"
m = adx.build_unet_denoiser(seed=cfg["seed"], **cfg["unet"])
adx.time_model_pass(m, cfg["T"], 3, prec, [0])
prof = adx.profile_model_pass(m, cfg["T"], prec, [0])
recs = prof.pop("records")
peak, _ = bench.load_peak("tensor", burst=True)
hbm, _ = bench.load_peak("hbm")
print(json.dumps(bench.per_launch_sol(recs, peak), indent=1))
t_sol = np.maximum(recs[:, 1] / (peak * 1e12), recs[:, 2] / (hbm * 1e9)) * 1e3
gap = recs[:, 3] - t_sol
names = {0: "conv", 1: "gemm", 2: "attn", 3: "gn", 4: "ln"}
print("largest gaps (ms above SOL): kind flops bytes ms sol_ms")
for i in np.argsort(-gap)[:25]:
    k, f, b, ms = recs[i]
    print(f"{names[int(k)]:5s} {f/1e9:9.2f} GF {b/1e6:8.2f} MB {ms*1e3:8.1f} us  sol {t_sol[i]*1e3:7.1f} us  "
          f"AI {f/b:7.1f}")
