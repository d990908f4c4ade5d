import os, sys, itertools
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
import paper_1311_7194_b200 as sf
base = bench.workload_config()
for rad, arc, sig, mode in itertools.product([0.25, 0.35], [0.3, 1.0], [4e-4, 0.0], [0, 2]):
    c = dict(base); c["orbit_radius"] = rad; c["orbit_arc"] = arc; c["sigma0"] = sig
    grid_cfg, intr, fusion, match = bench.make_params(sf, c)
    poses, frames = bench.make_frames(sf, c, 100, intr)
    hooks = bench.hook_deltas(sf, poses)
    g = sf.SparseTsdfGrid(grid_cfg, c["pool"], sf.AuxMode.Variance, p_min=c["p_min"])
    tr = sf.Tracker(g, intr, fusion, match, poses[0])
    lost, errs, its = None, [], []
    for k in range(100):
        tr.step(frames[k], mode, hooks[k])
        m = tr.fetch()
        if m.status:
            lost = k; break
        its.append(m.iterations)
        errs.append(max(np.abs(m.pose.translation - poses[k].translation).max(), np.abs(m.pose.rotation - poses[k].rotation).max()))
    print(f"rad={rad} arc={arc} sig={sig} mode={mode} lost_at={lost} max_err={max(errs):.2e} last_err={errs[-1]:.2e} "
          f"blocks={m.fusion.blocks_total} mean_it={np.mean(its):.1f} valid={(frames[0].depth>0).sum()}", flush=True)
    del tr, g
