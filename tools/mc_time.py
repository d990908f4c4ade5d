"""Marching cubes of a fused C4 volume: wall time of repeated extractions (device work + copy)."""
import sys
import time
sys.path.insert(0, '.')
import torch
import bench
import paper_1311_7194_b200 as sf
c = bench.workload_config()
g, intr, fusion, match = bench.make_params(sf, c)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
poses, frames = bench.make_frames(sf, c, n, intr)
grid = sf.SparseTsdfGrid(g, c["pool"], sf.AuxMode.Variance, p_min=c["p_min"])
for k in range(n):
    sf.fuse_frame(grid, frames[k], poses[k], fusion)
for it in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    v, nn, t = sf.marching_cubes(grid)
    print(f"mc: {len(t)} triangles {len(v)} vertices {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
