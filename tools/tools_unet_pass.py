"""One SD-2.1-shaped UNet pass for profiling: 3 warm-up + 1 timed pass (graph)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_06911_b200 as adx
m = adx.build_unet_denoiser(seed=0)
ms, b, n = adx.time_model_pass(m, 50, 1, "bf16", [0])
print("pass ms", ms)
