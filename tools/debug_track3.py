import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
import paper_1311_7194_b200 as sf
c = bench.workload_config(); c["orbit_arc"] = 1.0
for iters in [0, 15]:
    grid_cfg, intr, fusion, match = bench.make_params(sf, c)
    match.max_iterations = iters
    poses, frames = bench.make_frames(sf, c, 60, intr)
    hooks = bench.hook_deltas(sf, poses)
    g = sf.SparseTsdfGrid(grid_cfg, c["pool"], sf.AuxMode.Variance, p_min=c["p_min"])
    tr = sf.Tracker(g, intr, fusion, match, poses[0])
    out = []
    for k in range(60):
        tr.step(frames[k], 2, hooks[k])
        m = tr.fetch()
        R = m.pose.rotation
        orth = np.abs(R.T @ R - np.eye(3)).max()
        er = np.abs(R - poses[k].rotation).max(); et = np.abs(m.pose.translation - poses[k].translation).max()
        out.append(f"{k}:{m.status}/{er:.0e}/{et:.0e}/o{orth:.0e}/u{m.fusion.voxels_updated}")
        if m.status: break
    print(f"iters={iters}: " + " ".join(out), flush=True)
