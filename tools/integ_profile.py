"""Profiling driver (not a test): C4 bench frames fused at their ground-truth poses through the
stand-alone fuse_frame (plain launches, profilable by Nsight Compute), codes then float2."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_1311_7194_b200 as sfp
from paper_1311_7194_b200 import api as sf

n = int(sys.argv[1]) if len(sys.argv) > 1 else 12
layouts = sys.argv[2].split(",") if len(sys.argv) > 2 else ["codes", "float2"]
c = bench.workload_config()
grid_cfg, intr, fusion, _ = bench.make_params(sfp, c)
poses, frames = bench.make_frames(sfp, c, n, intr)
gpu = sf.default_backend()
for lay in layouts:
    g = sf.SparseTsdfGrid(grid_cfg, c["pool"], sf.AuxMode.Variance, p_min=c["p_min"])
    if lay == "float2":
        g.set_payload_layout(g.FLOAT2)
    for f, p in zip(frames, poses):
        st = gpu.fuse_frame(g, f, p, fusion)
    print(lay, st)
