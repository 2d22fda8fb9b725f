"""One UNet pass for profiling: 3 warm-up + 1 timed pass (graph).
usage: tools_unet_pass.py [bench config name, default c2] [precision, default bf16]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_06911_b200 as adx
from bench import CONFIGS
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
m = adx.build_unet_denoiser(seed=cfg["seed"], **cfg["unet"])
ms, b, n = adx.time_model_pass(m, cfg["T"], 1, sys.argv[2] if len(sys.argv) > 2 else "bf16", [0])
print("pass ms", ms)
