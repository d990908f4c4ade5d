import sys
sys.path.insert(0, '.')
import torch
import bench
import paper_1311_7194_b200 as sf
c = bench.workload_config()
g, intr, fusion, match = bench.make_params(sf, c)
poses, frames = bench.make_frames(sf, c, 40, intr)
dev = torch.device("cuda", 0)
df = [sf.DepthFrame(intr, torch.from_numpy(f.depth).to(dev), torch.from_numpy(f.sigma).to(dev)) for f in frames]
grid = sf.SparseTsdfGrid(g, c["pool"], sf.AuxMode.Variance, p_min=c["p_min"])
tr = sf.Tracker(grid, intr, fusion, match, poses[0])
hooks = bench.hook_deltas(sf, poses)
sp = torch.cuda.current_stream().cuda_stream
rows = []
for k in range(40):
    if bench.reseed_due(c, k):
        tr.set_pose(poses[k - 1], stream=sp)
    tr.step(df[k], sf.Tracker.TRACK_WITH_HOOK, hooks[k], stream=sp)
    m = tr.fetch(stream=sp)
    st = tr.stage_times()
    rows.append((m.iterations, st[1], st[0], st[4], m.kernel_launches))
from collections import defaultdict
agg = defaultdict(list)
for it, icp, rc, tot, nl in rows[5:]:
    agg[it].append(icp)
for it in sorted(agg):
    v = agg[it]
    print(f"iterations {it}: frames {len(v)} icp stage mean {1000*sum(v)/len(v):.1f} us")
