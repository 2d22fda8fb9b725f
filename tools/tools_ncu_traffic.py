"""DRAM traffic per UNet pass of each kernel family, from an ncu metrics capture of
tools/tools_unet_pass.py (4 graph replays of one pass: 3 warm-up + 1 timed), for the
`roofline.traffic` field of bench.py.  ncu flushes caches before each replayed kernel,
so these are cold-cache bytes per launch (an upper bound on what the kernel moves
inside the warm graph).
usage: tools_ncu_traffic.py launches.csv passes > profiles/r01_c2_dram_traffic.json"""
import csv
import json
import sys
from collections import defaultdict

path, passes = sys.argv[1], int(sys.argv[2])
rows = []
with open(path) as f:
    lines = [ln for ln in f if ln.startswith('"')]
for r in csv.DictReader(lines):
    rows.append(r)
fam = defaultdict(lambda: {"launches": 0, "dram_read": 0.0, "dram_write": 0.0, "ns": 0.0})
byid = defaultdict(dict)
for r in rows:
    byid[(r["ID"], r["Kernel Name"])][r["Metric Name"]] = (float(r["Metric Value"].replace(",", "")), r["Metric Unit"])
scale = {"ns": 1.0, "us": 1e3, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1.0, "usecond": 1e3, "msecond": 1e6}
for (kid, name), m in byid.items():
    short = name.replace("(anonymous namespace)::", "").replace("<unnamed>::", "").replace("unnamed>::", "").replace("void ", "")
    short = short.split("(")[0].split("<")[0].strip()
    d = fam[short]
    d["launches"] += 1
    v, u = m.get("dram__bytes_read.sum", (0.0, "byte"))
    d["dram_read"] += v * scale[u]
    v, u = m.get("dram__bytes_write.sum", (0.0, "byte"))
    d["dram_write"] += v * scale[u]
    v, u = m.get("gpu__time_duration.sum", (0.0, "nsecond"))
    d["ns"] += v * scale[u]
out = {}
for k, d in sorted(fam.items(), key=lambda kv: -kv[1]["ns"]):
    out[k] = {"launches_per_pass": d["launches"] / passes,
              "dram_bytes_per_pass": (d["dram_read"] + d["dram_write"]) / passes,
              "dram_read_per_pass": d["dram_read"] / passes, "dram_write_per_pass": d["dram_write"] / passes,
              "ncu_ms_per_pass": d["ns"] / passes * 1e-6}
print(json.dumps({"source": path, "passes": passes, "cache": "ncu default (flushed before each launch: cold)",
                  "families": out}, indent=1))
