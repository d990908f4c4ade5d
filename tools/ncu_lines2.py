"""Stall samples and executed instructions per CUDA source line (the cuda,sass view of an
.ncu-rep; line rows carry the aggregated metrics). usage: ncu_lines2.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, lines = "", []
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 8 and r[0].isdigit():  # a CUDA source line with aggregated metrics
        try:
            stall, inst = float(r[4] or 0), float(r[7] or 0)
        except ValueError:
            continue
        lines.append((stall, inst, f"{fname}:{r[0]}", r[1].strip()[:80]))
tot = sum(x[0] for x in lines) or 1
for st, ins, where, txt in sorted(lines, key=lambda x: -x[0])[:top]:
    print(f"{st / tot * 100:5.1f}% stall {ins:10.0f} inst  {where:22s} {txt}")
