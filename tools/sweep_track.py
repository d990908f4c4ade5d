"""Tracking-stability sweep of the C4 workload on the GPU tracker (same algorithm as the reference)."""
import os, sys, itertools
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
import paper_1311_7194_b200 as sf

c = bench.workload_config()
grid_cfg, intr, fusion, match0 = bench.make_params(sf, c)
poses, frames = bench.make_frames(sf, c, 100, intr)
hooks = bench.hook_deltas(sf, poses)
for mode, theta, maxd in itertools.product([2, 0], [0.005, 0.02, 0.05, 0.1], [4e-3, 1.5e-3]):
    match = bench.make_params(sf, c)[3]
    match.eigen_threshold = theta
    match.max_distance = maxd
    g = sf.SparseTsdfGrid(grid_cfg, c["pool"], sf.AuxMode.Variance, p_min=c["p_min"])
    tr = sf.Tracker(g, intr, fusion, match, poses[0])
    lost, errs = None, []
    for k in range(100):
        tr.step(frames[k], mode, hooks[k])
        m = tr.fetch()
        if m.status:
            lost = k
            break
        errs.append(max(np.abs(m.pose.translation - poses[k].translation).max(),
                        np.abs(m.pose.rotation - poses[k].rotation).max()))
    print(f"mode={mode} theta={theta} maxd={maxd} lost_at={lost} max_err={max(errs):.2e} last_err={errs[-1]:.2e} "
          f"blocks={m.fusion.blocks_total} it={m.iterations}", flush=True)
    del tr, g
