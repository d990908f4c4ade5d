"""Shared-memory bank conflicts per SASS instruction of one kernel in an .ncu-rep (source page):
excess wavefronts (L1 Wavefronts Shared Excessive) mapped to source lines. usage: ncu_smem.py rep kernel"""
import csv, io, subprocess, sys, collections
rep, kern = sys.argv[1], sys.argv[2]
def page(view):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kern,
                          "--launch-count", "1", "--print-source", view], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))
amap, cur, fname = {}, None, None
for r in page("cuda,sass"):
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if len(r) >= 4 and r[0] not in ("", "Line No", "Function Name"):
        cur = (fname, int(r[0]), r[1].strip()[:80])
    elif len(r) >= 4 and r[0] == "" and r[2].startswith("0x"):
        amap[r[2]] = cur
rows = page("sass")
hdr = next(r for r in rows if r and r[0] == "Address")
ix = {h: i for i, h in enumerate(hdr)}
acc = collections.Counter(); tot = collections.Counter()
for r in rows:
    if len(r) != len(hdr) or not r[0].startswith("0x"): continue
    num = lambda v: float(v) if v.replace(".", "", 1).isdigit() else 0.0
    ex = num(r[ix["L1 Wavefronts Shared Excessive"]]); wf = num(r[ix["L1 Wavefronts Shared"]])
    if wf == 0: continue
    key = amap.get(r[0], ("?", 0, r[1][:60]))
    acc[key] += ex; tot[key] += wf
print(f"total shared wavefronts {sum(tot.values()):.0f}, excessive {sum(acc.values()):.0f}")
for k, v in sorted(acc.items(), key=lambda x: -x[1])[:15]:
    print(f"{v:10.0f} excess of {tot[k]:10.0f}  {k[0]}:{k[1]}  {k[2]}")
