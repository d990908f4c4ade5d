"""Timing driver (not a test): the bench's C4 tracked sequence; per frame ICP steps, the ICP
device span (first step start .. last solve end) and the in-graph stage times (us)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
import paper_1311_7194_b200 as sfp
from paper_1311_7194_b200 import api as sf

steps, warm = int(os.environ.get("STEPS", "30")), 5
mode = os.environ.get("MODE", "hook")
c = bench.workload_config()
grid_cfg, intr, fusion, match = bench.make_params(sfp, c)
n = 1 + warm + steps
poses, frames = bench.make_frames(sfp, c, n, intr)
hooks = bench.hook_deltas(sfp, poses)
dev = torch.device("cuda", 0)
df = [sf.DepthFrame(intr, torch.from_numpy(f.depth).to(dev), torch.from_numpy(f.sigma).to(dev)) for f in frames]
flush = torch.empty(400 << 20, dtype=torch.uint8, device=dev)
sp = torch.cuda.current_stream().cuda_stream
H = sf.Tracker.TRACK_WITH_HOOK if mode == "hook" else sf.Tracker.TRACK
g = sf.SparseTsdfGrid(grid_cfg, c["pool"], sf.AuxMode.Variance, p_min=c["p_min"])
tr = sf.Tracker(g, intr, fusion, match, poses[0])
tr.set_stage_timing(int(os.environ.get("STAGES", "1")))
for k in range(1 + warm):
    if bench.reseed_due(c, k):
        tr.set_pose(poses[k - 1], stream=sp)
    tr.step(df[k], H, hooks[k] if mode == "hook" else None, stream=sp)
tr.fetch(stream=sp)
rows = []
for i in range(steps):
    k = 1 + warm + i
    if not os.environ.get("NOFLUSH"):
        flush.fill_(i & 255)
    if bench.reseed_due(c, k):
        tr.set_pose(poses[k - 1], stream=sp)
    tr.step(df[k], H, hooks[k] if mode == "hook" else None, stream=sp)
    m = tr.fetch(stream=sp)
    st = tr.stage_times()
    rows.append([m.icp_steps, m.icp_ns / 1e3] + [x * 1e3 for x in st])
a = np.array(rows)
for s in sorted(set(a[:, 0])):
    b = a[a[:, 0] == s]
    print(f"steps {int(s)}: frames {len(b)}, icp span {b[:,1].mean():.1f} us, stages " +
          " ".join(f"{x:.1f}" for x in b[:, 2:].mean(0)))
print("all: stages (raycast, icp, fuse prologue, integrate, total) " + " ".join(f"{x:.1f}" for x in a[:, 2:].mean(0)))
