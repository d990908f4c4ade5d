"""Sum an ncu_lines.py listing by source-line regions: ncu_regions.py <lines.txt> name:lo-hi ..."""
import re, sys
regs = []
for a in sys.argv[2:]:
    n, r = a.split(":"); lo, hi = r.split("-"); regs.append((n, int(lo), int(hi)))
tot = 0; acc = {}; samp = {}
for l in open(sys.argv[1]):
    m = re.match(r"\s*(\d+)\s+[\d.]+%\s+samples\s+([\d.]+)%\s+(\S+):(\d+)", l)
    if not m: continue
    n, s, f, ln = int(m.group(1)), float(m.group(2)), m.group(3), int(m.group(4))
    k = "other:" + f
    if f == "sf_fusion.cu":
        for name, lo, hi in regs:
            if lo <= ln <= hi: k = name; break
        else: k = "sf_fusion.cu other"
    acc[k] = acc.get(k, 0) + n; samp[k] = samp.get(k, 0) + s; tot += n
for k, v in sorted(acc.items(), key=lambda x: -x[1]):
    print(f"{k:28s} {v:10d} {100*v/tot:5.1f}%  stall {samp[k]:5.1f}%")
print("total", tot)
