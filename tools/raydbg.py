import sys, numpy as np
sys.path.insert(0, '.')
import bench
import paper_1311_7194_b200 as sf
c = bench.workload_config()
g, intr, fusion, match = bench.make_params(sf, c)
poses, frames = bench.make_frames(sf, c, 12, intr)
grid = sf.SparseTsdfGrid(g, c["pool"], sf.AuxMode.Variance, p_min=c["p_min"])
for k in range(12):
    sf.fuse_frame(grid, frames[k], poses[k], fusion)
d, n, st = sf.raycast_result(grid, poses[11], intr)
print(st)
