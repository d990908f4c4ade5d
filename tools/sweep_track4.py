import os, sys, itertools
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
import paper_1311_7194_b200 as sf
base = bench.workload_config()
for fmode, pmin, ped, qv in itertools.product(["kalman", "weighted"], [1e-12, 1e-8], [False, True], [-1.0, 1e-10]):
    if fmode == "weighted" and (pmin != 1e-12 or qv > 0):
        continue
    c = dict(base); c["orbit_arc"] = 1.0
    grid_cfg, intr, fusion, match = bench.make_params(sf, c)
    if fmode == "weighted":
        fusion = sf.FusionParams(mode=sf.FusionMode.Weighted, sigma0=c["sigma0"]); aux = sf.AuxMode.Weight
    else:
        aux = sf.AuxMode.Variance
        fusion.process_variance = qv
    poses = sf.orbit_trajectory(list(c["center"]), c["orbit_radius"], 100, (0.0, 1.0, 0.0), 0.0, 1.0)
    sc = bench.make_scene(sf, c)
    if ped:
        sc.add_box([0.0, -0.1, 0.35], [0.07, 0.02, 0.07])
    frames = [sf.render_synthetic_depth(sc, p, intr, sigma0=c["sigma0"], seed=1000 + k, domain_size=c["box_side"]) for k, p in enumerate(poses)]
    g = sf.SparseTsdfGrid(grid_cfg, c["pool"], aux, p_min=pmin)
    tr = sf.Tracker(g, intr, fusion, match, poses[0])
    lost, errs = None, []
    for k in range(100):
        tr.step(frames[k], 0)
        m = tr.fetch()
        if m.status:
            lost = k; break
        errs.append(max(np.abs(m.pose.translation - poses[k].translation).max(), np.abs(m.pose.rotation - poses[k].rotation).max()))
    print(f"{fmode} pmin={pmin} q={qv} ped={ped} lost_at={lost} max_err={max(errs):.2e} err@10={errs[10]:.2e} err@20={errs[20]:.2e}", flush=True)
    del tr, g
