cat > /tmp/gnp.py <<'PY'
import os, sys, subprocess, re, collections
sys.path.insert(0, os.getcwd())
code = r'''
import sys, os
sys.path.insert(0, os.getcwd())
import paper_2406_06911_b200 as adx
from bench import CONFIGS
cfg = CONFIGS["c5"]
m = adx.build_unet_denoiser(seed=cfg["seed"], **cfg["unet"])
adx.profile_model_pass(m, cfg["T"], "bf16")
'''
err = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, ADX_TC_TRACE="1"), capture_output=True, text=True).stderr
rows = [(float(a), float(b)) for a, b in re.findall(r"prof kind=3 ([\d.]+) us ([\d.]+) GB/s", err)]
agg = collections.defaultdict(lambda: [0, 0.0])
for i, (us, gbs) in enumerate(rows):
    bytes_ = gbs * us * 1e6
    key = ("stats" if bytes_ < 0 else "?", round(bytes_ / 1e6, 1))
    agg[round(bytes_ / 1e6, 1)][0] += 1; agg[round(bytes_ / 1e6, 1)][1] += us
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:8.1f} MB  {v[0]:3d} launches  {v[1]:8.1f} us  avg {v[1]/v[0]:6.1f} us  {k*1e3/(v[1]/v[0]):7.1f} GB/s")
PY
python /tmp/gnp.py
