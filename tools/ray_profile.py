"""Profiling driver (not a test): a C4 volume fused from the bench's first K frames (ground-truth
poses), then the raycast of frame K's pose through the plain sf_raycast launches
(k_ray_bounds, k_raycast, k_raycast_refine), timed with CUDA events over R repetitions."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1311_7194_b200 as sfp
from paper_1311_7194_b200 import api as sf

K = int(sys.argv[1]) if len(sys.argv) > 1 else 12
R = int(sys.argv[2]) if len(sys.argv) > 2 else 20
c = bench.workload_config()
grid_cfg, intr, fusion, _ = bench.make_params(sfp, c)
poses, frames = bench.make_frames(sfp, c, K + 1, intr)
gpu = sf.default_backend()
g = sf.SparseTsdfGrid(grid_cfg, c["pool"], sf.AuxMode.Variance, p_min=c["p_min"])
for f, p in zip(frames[:K], poses[:K]):
    gpu.fuse_frame(g, f, p, fusion)
dev = torch.device("cuda", 0)
d = torch.zeros((intr.height, intr.width), dtype=torch.float32, device=dev)
n = torch.zeros((intr.height, intr.width, 3), dtype=torch.float32, device=dev)
s = torch.cuda.current_stream()
flush = torch.empty(400 << 20, dtype=torch.uint8, device=dev)
ms = []
for r in range(R + 3):
    if not os.environ.get("NOFLUSH"):
        flush.fill_(r & 255)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    _, _, st = gpu.raycast_result(g, poses[K], intr, out_depth=d, out_normals=n, stream=s.cuda_stream)
    e1.record(s)
    torch.cuda.synchronize()
    if r >= 3:
        ms.append(e0.elapsed_time(e1))
ms.sort()
print(f"raycast: median {ms[len(ms)//2]*1e3:.1f} us, min {ms[0]*1e3:.1f} us; stats {st}")
if os.environ.get("SF_DIAG_RB"):
    import ctypes
    lib = ctypes.CDLL(os.environ["SF_GPU_LIB"])
    buf = (ctypes.c_ulonglong * 8)()
    lib.sf_debug_rb(buf)
    gpu.raycast_result(g, poses[K], intr, out_depth=d, out_normals=n, stream=s.cuda_stream)
    torch.cuda.synchronize()
    lib.sf_debug_rb(buf)
    print(f"DDA rays {buf[4]} (with bounds {buf[5]}): loop iterations before first occupied {buf[0]}, after {buf[1]}; "
          f"jumps before {buf[2]}, after {buf[3]}")
