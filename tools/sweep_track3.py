import os, sys, itertools
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
import paper_1311_7194_b200 as sf
base = bench.workload_config()
def scene_with(c, boxes):
    s = bench.make_scene(sf, c)
    for b in boxes:
        s.add_box(b[:3], b[3:])
    return s
variants = {
  "pedestal": [(0.0, -0.1, 0.35, 0.07, 0.02, 0.07)],
  "pedestal+block": [(0.0, -0.1, 0.35, 0.07, 0.02, 0.07), (0.06, -0.06, 0.30, 0.015, 0.02, 0.01)],
  "none": [],
}
for (name, boxes), arc, mode in itertools.product(variants.items(), [0.3, 1.0], [0, 2]):
    c = dict(base); c["orbit_arc"] = arc
    grid_cfg, intr, fusion, match = bench.make_params(sf, c)
    poses = sf.orbit_trajectory(list(c["center"]), c["orbit_radius"], 100, (0.0, 1.0, 0.0), 0.0, arc)
    sc = scene_with(c, boxes)
    frames = [sf.render_synthetic_depth(sc, p, intr, sigma0=c["sigma0"], seed=1000 + k, domain_size=c["box_side"]) for k, p in enumerate(poses)]
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
    print(f"{name} arc={arc} mode={mode} lost_at={lost} max_err={max(errs):.2e} err@10={errs[min(10,len(errs)-1)]:.2e} "
          f"blocks={m.fusion.blocks_total} mean_it={np.mean(its):.1f} valid={(frames[0].depth>0).sum()} upd={m.fusion.voxels_updated}", flush=True)
    del tr, g
