import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
import paper_1311_7194_b200 as sf
c = bench.workload_config(); c["orbit_arc"] = 1.0
grid_cfg, intr, fusion, match = bench.make_params(sf, c)
poses, frames = bench.make_frames(sf, c, 40, intr)
g = sf.SparseTsdfGrid(grid_cfg, c["pool"], sf.AuxMode.Variance, p_min=c["p_min"])
def perr(a, b):
    return np.abs(a.rotation - b.rotation).max(), np.abs(a.translation - b.translation).max()
for k in range(40):
    if k > 0:
        truth = sf.compose(sf.invert(poses[k - 1]), poses[k])
        d, n, _ = sf.raycast(g, poses[k - 1], intr)
        try:
            r = sf.icp(frames[k], d, n, truth, match)
            er, et = perr(r.delta, truth)
            s1 = f"model: it={r.iterations} m={r.matches} err_R={er:.1e} err_t={et:.1e} mask={''.join('1' if x else '0' for x in r.gated_mask)} lam/n={[round(x / r.pair_count, 4) for x in r.eigenvalues]}"
        except Exception as e:
            s1 = f"model: {type(e).__name__}"
        tn = sf.compute_normals(frames[k - 1], match.normal_sigma0, match.normal_spatial_scale)
        try:
            r2 = sf.icp(frames[k], frames[k - 1], tn, truth, match)
            er2, et2 = perr(r2.delta, truth)
            s2 = f"f2f: it={r2.iterations} m={r2.matches} err_R={er2:.1e} err_t={et2:.1e}"
        except Exception as e:
            s2 = f"f2f: {type(e).__name__}"
        if k % 3 == 1 or k > 24:
            print(f"k={k} {s1} | {s2}", flush=True)
    sf.fuse_frame(g, frames[k], poses[k], fusion)
