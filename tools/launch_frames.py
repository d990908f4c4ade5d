"""Per-frame kernel times of the bench's throughput run from an ncu launch-list CSV
(gpu__time_duration.sum): the launches between the (warmup+1)-th and the (warmup+steps)-th
k_integrate_rows of the first run, averaged per frame. Usage: launch_frames.py <csv> [warmup] [steps]"""
import collections
import csv
import sys

path = sys.argv[1]
warmup = int(sys.argv[2]) if len(sys.argv) > 2 else 5
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 60
rows = list(csv.reader(open(path)))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
data = [x for x in data if x["Metric Name"] == "gpu__time_duration.sum"]
idx = [i for i, x in enumerate(data) if "k_integrate_rows" in x["Kernel Name"]]
a, b = idx[warmup], idx[warmup + steps - 1]  # frame 0 is fused by the generic kernel
frames = steps - 1
agg, cnt = collections.defaultdict(float), collections.Counter()
for x in data[a + 1:b + 1]:
    if x["Kernel Name"].startswith(("at::", "void at::")):  # the bench's L2 flush (outside the timed steps)
        continue
    v = float(x["Metric Value"].replace(",", ""))
    u = x["Metric Unit"]
    v = v / 1000 if u in ("ns", "nsecond") else v * 1000 if u in ("ms", "msecond") else v
    k = x["Kernel Name"].split("(")[0].replace("void ", "")[:44]
    agg[k] += v
    cnt[k] += 1
tot = sum(agg.values())
print(f"{'us/frame':>9} {'launches/frame':>15} {'share':>6}  kernel   ({frames} frames)")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1]):
    print(f"{v / frames:9.1f} {cnt[k] / frames:15.2f} {100 * v / tot:5.1f}%  {k}")
print(f"{tot / frames:9.1f} us/frame serialised (ncu launch list)")
