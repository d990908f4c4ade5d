import sys
sys.path.insert(0, '.')
import bench
import paper_1311_7194_b200 as sf
c = bench.workload_config()
g, intr, fusion, match = bench.make_params(sf, c)
poses, frames = bench.make_frames(sf, c, 20, intr)
grid = sf.SparseTsdfGrid(g, c["pool"], sf.AuxMode.Variance, p_min=c["p_min"])
for k in range(20):
    sf.fuse_frame(grid, frames[k], poses[k], fusion)
