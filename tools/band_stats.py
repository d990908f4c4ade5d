"""Analysis (not a test): how the band |T| <= delta is distributed over the processed blocks
of a C4 frame (bench workload), to size row / block level out-of-band skipping."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
import paper_1311_7194_b200 as sfp
from paper_1311_7194_b200 import api as sf
from tests import oracle_backends

ref = oracle_backends.reference()
c = bench.workload_config()
grid_cfg, intr, fusion, match = bench.make_params(sfp, c)
K = int(sys.argv[1]) if len(sys.argv) > 1 else 5
poses, frames = bench.make_frames(sfp, c, K + 1, intr, backend=ref)
r = sf.SparseTsdfGrid(grid_cfg, c["pool"], sf.AuxMode.Variance, p_min=c["p_min"], backend=ref)
for k in range(K):
    ref.fuse_frame(r, frames[k], poses[k], fusion)
alloc, upd = ref.select_update_blocks(r, frames[K], poses[K])
blocks = np.concatenate([alloc, upd]).astype(np.int64)
print("blocks", len(blocks), "alloc", len(alloc), "update", len(upd))
M, vox, delta = c["M"], c["voxel"], r.delta
org = np.array(c["box_origin"])
P = poses[K]
Rt = P.rotation.T
t = P.translation
l = np.arange(M)
lz, ly, lx = np.meshgrid(l, l, l, indexing="ij")  # [z][y][x]
loc = np.stack([lx, ly, lz], -1).reshape(-1, 3)  # voxel order x fastest
d = frames[K].depth
W, H = d.shape[1], d.shape[0]
inband = np.zeros((len(blocks), M ** 3), bool)
for s0 in range(0, len(blocks), 2000):
    b = blocks[s0:s0 + 2000]
    vc = (b[:, None, :] * M + loc[None]).astype(np.float64)
    x = org + (vc + 0.5) * vox
    xc = (x - t) @ Rt.T
    z = xc[..., 2]
    u = np.floor(525.0 * xc[..., 0] / z + 319.5 + 0.5).astype(np.int64)
    v = np.floor(525.0 * xc[..., 1] / z + 239.5 + 0.5).astype(np.int64)
    ok = (z > 0) & (u >= 0) & (v >= 0) & (u < W) & (v < H)
    dd = np.where(ok, d[np.clip(v, 0, H - 1), np.clip(u, 0, W - 1)], 0.0)
    T = dd - z
    inband[s0:s0 + 2000] = (dd > 0) & (np.abs(T) <= delta)
nv = inband.size
print(f"voxels {nv}, in band {inband.mean():.3f}")
rows = inband.reshape(len(blocks), M * M, M)  # [block][z*M+y][x]
print(f"x-rows with an in-band voxel: {rows.any(-1).mean():.3f}")
half = inband.reshape(len(blocks), 2, M ** 3 // 2)
print(f"32-row half blocks with an in-band voxel: {half.any(-1).mean():.3f}")
print(f"blocks with an in-band voxel: {inband.any(-1).mean():.3f}")
zsl = inband.reshape(len(blocks), M, M * M)
print(f"z slices (64 voxels) with an in-band voxel: {zsl.any(-1).mean():.3f}")
q = inband.reshape(len(blocks), M, M, M)
for name, ax in (("x", 3), ("y", 2), ("z", 1)):
    print(f"rows along {name} with in-band: {q.any(ax).mean():.3f}; in-band per such row {q.sum(ax)[q.any(ax)].mean():.2f}")

# pixel footprint of rows along each axis: distinct lround(u) / lround(v) per row
def footprint(axis):
    res = []
    for s0 in range(0, len(blocks), 2000):
        b = blocks[s0:s0 + 2000]
        vc = (b[:, None, :] * M + loc[None]).astype(np.float64)
        x = org + (vc + 0.5) * vox
        xc = (x - t) @ Rt.T
        u = np.floor(525.0 * xc[..., 0] / xc[..., 2] + 319.5 + 0.5)
        v = np.floor(525.0 * xc[..., 1] / xc[..., 2] + 239.5 + 0.5)
        u = u.reshape(len(b), M, M, M); v = v.reshape(len(b), M, M, M)   # [z][y][x]
        ax = {0: 3, 1: 2, 2: 1}[axis]
        cu = u.max(ax) - u.min(ax) + 1
        cv = v.max(ax) - v.min(ax) + 1
        res.append(np.stack([cu.reshape(-1), cv.reshape(-1)], -1))
    r = np.concatenate(res)
    return r
Rcam = P.rotation.T  # world -> camera rotation
for a in range(3):
    r = footprint(a)
    print(f"axis {'xyz'[a]} (cam z comp {Rcam[2, a]:+.3f}): rows with cols<=2 & rows<=2: {((r[:,0]<=2)&(r[:,1]<=2)).mean():.3f}, "
          f"single pixel {((r[:,0]==1)&(r[:,1]==1)).mean():.3f}, cols<=3&rows<=2 {((r[:,0]<=3)&(r[:,1]<=2)).mean():.3f}")
