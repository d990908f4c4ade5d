"""Per-instruction SASS listing with execution counts and stall samples from an .ncu-rep.
usage: python tools/ncu_sass.py report.ncu-rep > listing.txt"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ie, src, ws = h.index("Instructions Executed"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
tot = 0
for r in rows[2:]:
    try:
        v = float(r[ie])
    except (ValueError, IndexError):
        continue
    tot += v
    print(f"{v:9.0f} {r[ws]:>4} {r[src][:110]}")
print(f"# total warp instructions {tot:.0f}", file=sys.stderr)
