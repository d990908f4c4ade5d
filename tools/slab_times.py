"""Timing diagnostic (not a test): per-warp timeline of the last k_integrate_slab launch
(library built with -DSF_DIAG_TIMES=1): kernel entry, first unit, end, units processed."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
import paper_1311_7194_b200 as sfp
from paper_1311_7194_b200 import api as sf

n = int(sys.argv[1]) if len(sys.argv) > 1 else 12
c = bench.workload_config()
grid_cfg, intr, fusion, _ = bench.make_params(sfp, c)
poses, frames = bench.make_frames(sfp, c, n, intr)
gpu = sf.default_backend()
lib = ctypes.CDLL(os.environ["SF_GPU_LIB"])
for lay in sys.argv[2].split(",") if len(sys.argv) > 2 else ["codes", "float2"]:
    g = sf.SparseTsdfGrid(grid_cfg, c["pool"], sf.AuxMode.Variance, p_min=c["p_min"])
    if lay == "float2":
        g.set_payload_layout(g.FLOAT2)
    for f, p in zip(frames, poses):
        st = gpu.fuse_frame(g, f, p, fusion)
    W = 148 * 4 * 8
    buf = (ctypes.c_ulonglong * (4 * W))()
    assert lib.sf_debug_slab_times(buf, 4 * W) == 0
    a = np.frombuffer(buf, dtype=np.uint64).reshape(W, 4).astype(np.int64)
    a = a[a[:, 0] > 0]
    t0 = a[:, 0].min()
    e, f1, end, units = (a[:, 0] - t0) / 1e3, (a[:, 1] - t0) / 1e3, (a[:, 2] - t0) / 1e3, a[:, 3] & 0xFFFF
    last = e + (a[:, 3] >> 16) / 1e3
    q = lambda x: " ".join(f"{v:6.1f}" for v in np.percentile(x, [0, 10, 50, 90, 100]))
    print(f"{lay}: warps {len(a)}  (percentiles 0/10/50/90/100, us from first entry)")
    print(f"  entry      {q(e)}")
    print(f"  first unit {q(f1)}")
    print(f"  end        {q(end)}")
    print(f"  units      {q(units)}  total {units.sum()}")
    o = np.argsort(-end)[:12]
    print("  latest warps (gwarp: units, last unit start, end):",
          "; ".join(f"{int(i)}: {int(units[i])}, {last[i]:.1f}, {end[i]:.1f}" for i in o))
    busy = end - f1
    print(f"  busy/unit  {q(busy / np.maximum(units, 1))}")
