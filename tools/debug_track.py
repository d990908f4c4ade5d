"""Debug: per-frame tracker metrics on the C4 bench workload (GPU), optional reference check."""
import ctypes as C
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
import paper_1311_7194_b200 as sf
from paper_1311_7194_b200 import _abi as A

nref = int(sys.argv[1]) if len(sys.argv) > 1 else 0
mode = int(sys.argv[2]) if len(sys.argv) > 2 else 2
c = bench.workload_config()
grid_cfg, intr, fusion, match = bench.make_params(sf, c)
poses, frames = bench.make_frames(sf, c, 40, intr)
hooks = bench.hook_deltas(sf, poses)
g = sf.SparseTsdfGrid(grid_cfg, c["pool"], sf.AuxMode.Variance, p_min=c["p_min"])
tr = sf.Tracker(g, intr, fusion, match, poses[0])
ref = None
if nref:
    from tests import oracle_backends
    ref = oracle_backends.reference()
    rg = sf.SparseTsdfGrid(grid_cfg, c["pool"], sf.AuxMode.Variance, p_min=c["p_min"], backend=ref)
    cur = poses[0].to12().copy()
for k in range(40):
    tr.step(frames[k], mode, hooks[k])
    m = tr.fetch()
    gt = poses[k]
    err_t = float(np.abs(m.pose.translation - gt.translation).max())
    err_r = float(np.abs(m.pose.rotation - gt.rotation).max())
    print(f"k={k} status={m.status} it={m.iterations} matches={m.matches} rms={m.residual_rms:.3e} "
          f"hits={m.raycast.hit_pixels} rwb={m.raycast.rays_with_bounds} blocks={m.fusion.blocks_total} "
          f"proc={m.blocks_processed} upd={m.fusion.voxels_updated} err_t={err_t:.2e} err_r={err_r:.2e} "
          f"gated={''.join('1' if x else '0' for x in m.gated_mask)} valid={(frames[k].depth>0).sum()}", flush=True)
    if ref is not None and k < nref:
        st = A.FusionStatsC(); it = C.c_int32(); mt = C.c_uint64()
        fc, ic, fp, mp = frames[k].c(), intr.c(), fusion.c(), match.c()
        ext = hooks[k].to12()
        rc = ref.lib.pipeline_frame(rg.handle, C.byref(fc), C.byref(ic), C.byref(fp), C.byref(mp),
                                    1 if k == 0 else mode, ext.ctypes.data_as(A.c_double_p),
                                    cur.ctypes.data_as(A.c_double_p), C.byref(st), C.byref(it), C.byref(mt))
        rp = sf.Pose.from12(cur)
        print(f"   ref rc={rc} it={it.value} matches={mt.value} blocks={st.blocks_total} upd={st.voxels_updated} "
              f"dpose={max(np.abs(rp.rotation-m.pose.rotation).max(), np.abs(rp.translation-m.pose.translation).max()):.2e}",
              flush=True)
    if m.status:
        break
