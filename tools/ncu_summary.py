"""Summarise one kernel of an .ncu-rep: SOL, occupancy, stall reasons, instruction mix.
usage: python tools/ncu_summary.py report.ncu-rep [row]  (row: which launch of the report, default 0)"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, u, v = r[0], r[1], r[2 + (int(sys.argv[2]) if len(sys.argv) > 2 else 0)]
d = dict(zip(h, v))
units = dict(zip(h, u))
keys = ["Kernel Name", "gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__cycles_active.avg", "gpc__cycles_elapsed.max", "launch__registers_per_thread",
        "lts__t_sector_hit_rate.pct"]
for k in keys:
    print(f"{k:60s} {d.get(k, '?')[:120]} {units.get(k, '') if k != 'Kernel Name' else ''}")
st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(x.replace(",", "") or 0)
      for k, x in d.items() if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
tot = sum(st.values()) or 1
print("stalls:", ", ".join(f"{k} {v / tot * 100:.0f}%" for k, v in sorted(st.items(), key=lambda x: -x[1])[:8]))
pipes = {k.split("pipe_")[1].split(".")[0]: x for k, x in d.items()
         if k.startswith("sm__inst_executed_pipe_") and k.endswith("sum.pct_of_peak_sustained_active")}
print("pipes %:", ", ".join(f"{k} {x}" for k, x in sorted(pipes.items(), key=lambda x: -float(x[1] or 0))[:8]))
