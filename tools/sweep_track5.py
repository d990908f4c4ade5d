import os, sys, itertools
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
import paper_1311_7194_b200 as sf
base = bench.workload_config()
for arc, boot, mode in itertools.product([0.3, 1.0], [1, 5, 10], [2, 0]):
    c = dict(base); c["orbit_arc"] = arc
    grid_cfg, intr, fusion, match = bench.make_params(sf, c)
    poses, frames = bench.make_frames(sf, c, 100, intr)
    hooks = bench.hook_deltas(sf, poses)
    g = sf.SparseTsdfGrid(grid_cfg, c["pool"], sf.AuxMode.Variance, p_min=c["p_min"])
    tr = sf.Tracker(g, intr, fusion, match, poses[0])
    lost, errs = None, []
    for k in range(100):
        if k < boot:
            tr.step(frames[k], 1, poses[k])
        else:
            tr.step(frames[k], mode, hooks[k])
        m = tr.fetch()
        if m.status:
            lost = k; break
        errs.append(max(np.abs(m.pose.translation - poses[k].translation).max(), np.abs(m.pose.rotation - poses[k].rotation).max()))
    print(f"arc={arc} boot={boot} mode={mode} lost_at={lost} max_err={max(errs):.2e} err@30={errs[min(30,len(errs)-1)]:.2e} last={errs[-1]:.2e}", flush=True)
    del tr, g
