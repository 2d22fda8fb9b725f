"""Per-shape isolated launch times of one UNet pass (ADX_TC_TRACE=1 + profile_model_pass):
aggregates GEMM / conv / attention / norm launches by shape, sorted by total time.
usage: tools_shape_profile.py [bench config, default c2] [precision, default bf16]"""
import collections, os, re, subprocess, sys
HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 2 and sys.argv[2] == "--child":
    sys.path.insert(0, HERE)
    import paper_2406_06911_b200 as adx
    from bench import CONFIGS
    cfg = CONFIGS[sys.argv[1]]
    m = adx.build_unet_denoiser(seed=cfg["seed"], **cfg["unet"])
    adx.profile_model_pass(m, cfg["T"], sys.argv[3])
    sys.exit(0)
conf = sys.argv[1] if len(sys.argv) > 1 else "c2"
prec = sys.argv[2] if len(sys.argv) > 2 else "bf16"
err = subprocess.run([sys.executable, __file__, conf, "--child", prec], env=dict(os.environ, ADX_TC_TRACE="1"),
                     capture_output=True, text=True).stderr.splitlines()
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
last = None
for l in err:
    if l.startswith("tc_gemm") or l.startswith("tc_conv3x3") or l.startswith("tc_attention"):
        last = re.sub(r" grid=\S+", "", l.strip())
        continue
    p = re.match(r"\s*prof kind=(\d+) ([\d.]+) us ([\d.]+) (.*)", l)
    if p:
        kind, us, rate = int(p.group(1)), float(p.group(2)), float(p.group(3))
        key = last if kind in (0, 1, 2) and last else f"kind={kind} {p.group(4)}"
        agg[key][0] += 1
        agg[key][1] += us
        agg[key][2] = rate
        last = None
tot = sum(v[1] for v in agg.values())
print(f"{conf}: {sum(v[0] for v in agg.values())} launches, {tot / 1e3:.3f} ms isolated")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:40]:
    print(f"{v[1]:8.1f} us {v[0]:3d} x {v[1] / v[0]:6.1f}  {v[2]:7.1f} G/s|TF  {k}")
