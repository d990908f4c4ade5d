"""Timing diagnostic (not a test): the ICP step tail of the last tracked frame (library built with
-DSF_DIAG_ICP_TAIL for sf_icp.cu and -DSF_DIAG_ICP_ASSOC for sf_tracker.cu)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1311_7194_b200 as sfp
from paper_1311_7194_b200 import api as sf

c = bench.workload_config()
grid_cfg, intr, fusion, match = bench.make_params(sfp, c)
poses, frames = bench.make_frames(sfp, c, 12, intr)
hooks = bench.hook_deltas(sfp, poses)
dev = torch.device("cuda", 0)
df = [sf.DepthFrame(intr, torch.from_numpy(f.depth).to(dev), torch.from_numpy(f.sigma).to(dev)) for f in frames]
sp = torch.cuda.current_stream().cuda_stream
g = sf.SparseTsdfGrid(grid_cfg, c["pool"], sf.AuxMode.Variance, p_min=c["p_min"])
tr = sf.Tracker(g, intr, fusion, match, poses[0])
lib = ctypes.CDLL(os.environ["SF_GPU_LIB"])
for k in range(12):
    if bench.reseed_due(c, k):
        tr.set_pose(poses[k - 1], stream=sp)
    tr.step(df[k], sf.Tracker.TRACK_WITH_HOOK, hooks[k], stream=sp)
    m = tr.fetch(stream=sp)
    buf = (ctypes.c_ulonglong * 8)()
    lib.sf_debug_icp_tail(buf)
    t = [buf[i] - buf[0] for i in range(5)]
    print(f"frame {k}: steps {m.icp_steps} assoc {m.icp_ns/1e3:.1f} us | tail from last-CTA: sums {t[1]/1e3:.1f}, "
          f"L-map {t[2]/1e3:.1f}, chol {t[3]/1e3:.1f}, motion {t[4]/1e3:.1f} us")
