"""Diagnostic (not a test): one ICP call at the bench's C4 workload on identical inputs, GPU vs
the reference build, per max_iterations — pose difference, match counts, iterations."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
import paper_1311_7194_b200 as sfp
from paper_1311_7194_b200 import api as sf
from tests import oracle_backends

ref = oracle_backends.reference()
gpu = sf.default_backend()
c = bench.workload_config()
grid_cfg, intr, fusion, match = bench.make_params(sfp, c)
poses, frames = bench.make_frames(sfp, c, 6, intr)
hooks = bench.hook_deltas(sfp, poses)
g = sf.SparseTsdfGrid(grid_cfg, c["pool"], sf.AuxMode.Variance, p_min=c["p_min"], backend=gpu)
r = sf.SparseTsdfGrid(grid_cfg, c["pool"], sf.AuxMode.Variance, p_min=c["p_min"], backend=ref)
for k in range(4):
    gpu.fuse_frame(g, frames[k], poses[k], fusion)
    ref.fuse_frame(r, frames[k], poses[k], fusion)
print("tables equal", np.array_equal(g.read_table(), r.read_table()))
dg, ng, _ = gpu.raycast(g, poses[3], intr)
dr, nr, _ = ref.raycast(r, poses[3], intr)
print("raycast equal", np.array_equal(dg.depth, dr.depth), np.array_equal(ng.array, nr.array))
init = hooks[4]
for mi in [1, 2, 3, 4, 6, 15]:
    m = sf.MatchParams.for_voxel_size(grid_cfg.voxel_size)
    m.max_distance = match.max_distance
    m.normal_sigma0 = match.normal_sigma0
    m.max_iterations = mi
    a = gpu.icp(frames[4], dr, nr, init, m)
    b = ref.icp(frames[4], dr, nr, init, m)
    d = np.abs(a.delta.to12() - b.delta.to12()).max()
    print(f"max_it {mi}: it {a.iterations}/{b.iterations} matches {a.matches}/{b.matches} pose diff {d:.3e}")
