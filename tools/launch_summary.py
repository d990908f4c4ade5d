"""Summarise an ncu launch-list CSV (gpu__time_duration.sum) over the last N launches."""
import collections
import csv
import sys

path = sys.argv[1]
last = int(sys.argv[2]) if len(sys.argv) > 2 else 350
rows = list(csv.reader(open(path)))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
data = [x for x in data if x["Metric Name"] == "gpu__time_duration.sum"][-last:]
agg = collections.defaultdict(lambda: [0, 0.0, []])
for x in data:
    v = float(x["Metric Value"].replace(",", ""))
    v = {"ns": v / 1000, "nsecond": v / 1000, "us": v, "usecond": v, "ms": v * 1000, "msecond": v * 1000}[x["Metric Unit"]]
    a = agg[x["Kernel Name"].split("(")[0][:48]]
    a[0] += 1
    a[1] += v
    a[2].append(v)
tot = sum(a[1] for a in agg.values())
print(f"{'total_us':>9} {'n':>4} {'mean_us':>8} {'max_us':>8} {'share':>6}  kernel")
for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{a[1]:9.1f} {a[0]:4d} {a[1] / a[0]:8.1f} {max(a[2]):8.1f} {100 * a[1] / tot:5.1f}%  {k}")
print(f"{tot:9.1f} us total over {len(data)} launches")
