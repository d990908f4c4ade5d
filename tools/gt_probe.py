import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
import paper_1311_7194_b200 as sf
c = bench.workload_config()
for variant in ["base", "nonoise", "weighted"]:
    cc = dict(c)
    if variant == "nonoise":
        cc["sigma0"] = 0.0
    grid_cfg, intr, fusion, match = bench.make_params(sf, cc)
    poses, frames = bench.make_frames(sf, cc, 60, intr)
    aux = sf.AuxMode.Variance
    if variant == "weighted":
        fusion = sf.FusionParams(mode=sf.FusionMode.Weighted, sigma0=cc["sigma0"])
        aux = sf.AuxMode.Weight
    g = sf.SparseTsdfGrid(grid_cfg, cc["pool"], aux, p_min=cc["p_min"])
    tr = sf.Tracker(g, intr, fusion, match, poses[0])
    out = []
    for k in range(60):
        tr.step(frames[k], 1, poses[k])
        m = tr.fetch()
        if k % 4 == 0 or k > 22 and k < 34:
            d, n, st = sf.raycast_result(g, poses[k], intr)
            out.append(f"k={k}:proc={m.blocks_processed},upd={m.fusion.voxels_updated},blk={m.fusion.blocks_total},hits={st.hit_pixels}")
    print(variant, " | ".join(out), flush=True)
