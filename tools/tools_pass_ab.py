"""UNet pass time (graph of back-to-back passes, CUDA events) for the library variants named on
the command line (ADX_LIB_VARIANT; '-' = the product build), each in its own process.
usage: tools_pass_ab.py [--configs c2,c4,c5] variant ..."""
import os, subprocess, sys
args = sys.argv[1:]
configs = ["c2"]
if args and args[0] == "--configs":
    configs = args[1].split(","); args = args[2:]
code = r'''
import sys, os
sys.path.insert(0, os.getcwd())
import paper_2406_06911_b200 as adx
from bench import CONFIGS
for c in sys.argv[1].split(","):
    cfg = CONFIGS[c]
    m = adx.build_unet_denoiser(seed=cfg["seed"], **cfg["unet"])
    adx.time_model_pass(m, cfg["T"], 3, "bf16", [0])
    best = min(adx.time_model_pass(m, cfg["T"], 10, "bf16", [0])[0] for _ in range(3))
    print(c, "pass ms", round(best, 4), flush=True)
    del m
'''
for v in args:
    env = dict(os.environ)
    if v != "-":
        env["ADX_LIB_VARIANT"] = v
    out = subprocess.run([sys.executable, "-c", code, ",".join(configs)], env=env, capture_output=True, text=True)
    print("==", v, out.stdout.strip().replace("\n", " | "), out.stderr.strip()[-300:] if out.returncode else "", flush=True)
