import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
import paper_1311_7194_b200 as sf
c = bench.workload_config(); c["orbit_arc"] = 1.0
grid_cfg, intr, fusion, match = bench.make_params(sf, c)
poses, frames = bench.make_frames(sf, c, 60, intr)
hooks = bench.hook_deltas(sf, poses)
g = sf.SparseTsdfGrid(grid_cfg, c["pool"], sf.AuxMode.Variance, p_min=c["p_min"])
tr = sf.Tracker(g, intr, fusion, match, poses[0])
for k in range(60):
    tr.step(frames[k], 1 if k < 10 else 2, poses[k] if k < 10 else hooks[k])
    m = tr.fetch()
    st = tr.stage_times()
    er = np.abs(m.pose.rotation - poses[k].rotation).max(); et = np.abs(m.pose.translation - poses[k].translation).max()
    if k >= 8:
        print(f"k={k} st={m.status} it={m.iterations} m={m.matches} rms={m.residual_rms:.2e} hits={m.raycast.hit_pixels} "
              f"steps={m.raycast.sample_steps} proc={m.blocks_processed} blk={m.fusion.blocks_total} upd={m.fusion.voxels_updated} "
              f"eR={er:.1e} et={et:.1e} lam={[round(x,3) for x in m.lambda_over_n]} ms={[round(x,3) for x in st]}", flush=True)
    if m.status: break
