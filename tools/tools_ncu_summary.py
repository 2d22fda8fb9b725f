"""Key metrics of every kernel in an ncu --set full report (for profiles/*_ncu_full_summary.txt).
usage: tools_ncu_summary.py report.ncu-rep"""
import csv, io, subprocess, sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "l1tex__m_xbar2l1tex_read_bytes.sum", "sm__cycles_active.avg", "sm__cycles_elapsed.avg",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__grid_size", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic"]
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, body = rows[0], rows[2:]
for r in body:
    d = dict(zip(hdr, r))
    print(d.get("Kernel Name", "?").split("(")[0].replace("void ", ""))
    for k in KEYS:
        if k in d:
            print(f"    {k} = {d[k]}")
    stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): d[k] for k in d
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
    top = sorted(((float(v), k) for k, v in stalls.items() if v.replace(".", "", 1).isdigit()), reverse=True)[:5]
    print("    top stall samples: " + ", ".join(f"{k} {int(v)}" for v, k in top))
