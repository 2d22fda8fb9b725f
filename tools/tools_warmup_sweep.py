"""Warm-up sweep (experiment.cpp:312-389 analogue) on the c2 UNet: async trajectory vs the
sequential one for N in {2, 3, 4} x w in {1, 2, 3, 5, 9, 15} (S=1) and N=3 S=2 -- the paper's
Table-2 analogue.  usage: tools_warmup_sweep.py [out.json]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_06911_b200 as adx
from oracle import oracle as O
from bench import CONFIGS

cfg = CONFIGS["c2"]
m = adx.build_unet_denoiser(seed=cfg["seed"], **cfg["unet"])
s = adx.build_schedule(cfg["T"], cfg["beta"][0], cfg["beta"][1], "linear")
x = adx.Latent(O.random_normals(cfg["x_seed"], m.data_dim()), cfg["T"])
matrix = [(N, w, 1) for N in (2, 3, 4) for w in (1, 2, 3, 5, 9, 15)] + [(3, w, 2) for w in (3, 9)]
rows = adx.warmup_sweep(m, x, s, matrix, precision="bf16")
for r in rows:
    print(json.dumps(r), flush=True)
json.dump(dict(config="c2 (SD-2.1-shaped UNet, 96x96x4, T=50, bf16)", rows=rows),
          open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/warmup_sweep.json", "w"), indent=1)
