"""Join an ncu SASS source page (per-instruction counts) with its cuda,sass page (address ->
source line) and print the hottest source lines. Usage:
  ncu_lines.py <report.ncu-rep> <kernel-regex> [launch-skip] [top]"""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40


def page(view):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kern,
                          "--launch-skip", skip, "--launch-count", "1", "--print-source", view],
                         capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


amap, cur, fname = {}, None, None
for r in page("cuda,sass"):
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) >= 4 and r[0] not in ("", "Line No", "Function Name"):
        cur = (fname, int(r[0]), r[1].strip()[:80])
    elif len(r) >= 4 and r[0] == "" and r[2].startswith("0x"):
        amap[r[2]] = cur
rows = page("sass")
h = rows[1]
iA, iE, iS = h.index("Address"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
agg = collections.defaultdict(lambda: [0, 0])
tot = tots = 0
for r in rows[2:]:
    if len(r) <= max(iE, iS) or not r[iE].isdigit():
        continue
    k = amap.get(r[iA], ("?", 0, ""))
    agg[k][0] += int(r[iE])
    agg[k][1] += int(r[iS])
    tot += int(r[iE])
    tots += int(r[iS])
print(f"total warp instructions {tot}, stall samples {tots}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{v[0]:10d} {100 * v[0] / tot:5.1f}%  samples {100 * v[1] / max(tots, 1):5.1f}%  {k[0]}:{k[1]}  {k[2]}")
