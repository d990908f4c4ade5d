"""Timing driver (not a test): the bench's C4 tracked sequence (icp_with_hook, relocalised) with
the in-graph stage events, mean stage times in us: raycast, icp, fuse prologue, integrate, total."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1311_7194_b200 as sfp
from paper_1311_7194_b200 import api as sf

steps, warm = int(os.environ.get("STEPS", "20")), 5
c = bench.workload_config()
grid_cfg, intr, fusion, match = bench.make_params(sfp, c)
n = 1 + warm + steps
poses, frames = bench.make_frames(sfp, c, n, intr)
hooks = bench.hook_deltas(sfp, poses)
dev = torch.device("cuda", 0)
df = [sf.DepthFrame(intr, torch.from_numpy(f.depth).to(dev), torch.from_numpy(f.sigma).to(dev)) for f in frames]
flush = torch.empty(400 << 20, dtype=torch.uint8, device=dev)
sp = torch.cuda.current_stream().cuda_stream
H = sf.Tracker.TRACK_WITH_HOOK
for rep in range(int(os.environ.get("REPS", "1"))):
    g = sf.SparseTsdfGrid(grid_cfg, c["pool"], sf.AuxMode.Variance, p_min=c["p_min"])
    tr = sf.Tracker(g, intr, fusion, match, poses[0])
    tr.set_stage_timing(2)
    for k in range(1 + warm):
        if bench.reseed_due(c, k):
            tr.set_pose(poses[k - 1], stream=sp)
        tr.step(df[k], H, hooks[k], stream=sp)
    tr.fetch(stream=sp)
    acc = [0.0] * 5
    for i in range(steps):
        k = 1 + warm + i
        flush.fill_(i & 255)
        if bench.reseed_due(c, k):
            tr.set_pose(poses[k - 1], stream=sp)
        tr.step(df[k], H, hooks[k], stream=sp)
        m = tr.fetch(stream=sp)
        st = tr.stage_times()
        acc = [a + b for a, b in zip(acc, st)]
    print("stages us:", " ".join(f"{x * 1e3 / steps:.1f}" for x in acc), "| pose", m.pose.to12()[9:].round(9))
