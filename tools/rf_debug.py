"""Per-ray timing of the refine pass (stage 2 + normal) on the C4 bench sequence (debug aid)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1311_7194_b200 as sf  # noqa: E402

FIRST = int(sys.argv[1]) if len(sys.argv) > 1 else 40
out = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/rf_debug.bin"
c = bench.workload_config()
grid_cfg, intr, fusion, match = bench.make_params(sf, c)
poses, frames = bench.make_frames(sf, c, FIRST + 2, intr)
dev = torch.device("cuda", 0)
dframes = [sf.DepthFrame(intr, torch.from_numpy(f.depth).to(dev), torch.from_numpy(f.sigma).to(dev)) for f in frames]
grid = sf.SparseTsdfGrid(grid_cfg, c["pool"], sf.AuxMode.Variance, p_min=c["p_min"], device=0)
tr = sf.Tracker(grid, intr, fusion, match, poses[0], use_graphs=False)
hooks = bench.hook_deltas(sf, poses)
sp = torch.cuda.current_stream().cuda_stream
if os.path.exists(out):
    os.remove(out)
for k in range(FIRST + 2):
    if k >= FIRST:
        os.environ["SF_RF_DEBUG"] = out
    if bench.reseed_due(c, k) and k > 0:
        tr.set_pose(poses[k - 1], stream=sp)
    tr.step(dframes[k], sf.Tracker.TRACK_WITH_HOOK, hooks[k], stream=sp)
    tr.fetch(stream=sp)
os.environ.pop("SF_RF_DEBUG", None)
raw = np.fromfile(out, dtype=np.uint64)
pos = 0
while pos < len(raw):
    nb = int(raw[pos])
    d = raw[pos + 1:pos + 1 + 4 * nb].reshape(nb, 4).astype(np.int64)
    pos += 1 + 4 * nb
    t0, tm, t1 = d[:, 0], d[:, 1], d[:, 2]
    it = d[:, 3] & 0xFFFFFFFF
    base = t0.min()
    print(f"brackets {nb}: span {(t1.max() - base) / 1e3:.1f} us; start spread {(t0.max() - base) / 1e3:.1f} us")
    print("  iterations percentiles 50/90/99/max:", [int(np.percentile(it, q)) for q in (50, 90, 99, 100)],
          "mean", round(float(it.mean()), 2), " rays at 48:", int((it >= 48).sum()))
    sec = (tm - t0) / 1e3
    grad = (t1 - tm) / 1e3
    print("  secant us p50/p90/p99/max:", [round(float(np.percentile(sec, q)), 2) for q in (50, 90, 99, 100)])
    print("  gradient us p50/p90/p99/max:", [round(float(np.percentile(grad, q)), 2) for q in (50, 90, 99, 100)])
    for lo, hi in ((0, 4), (4, 8), (8, 16), (16, 32), (32, 48), (48, 49)):
        m = (it >= lo) & (it < hi)
        if m.any():
            print(f"   iters [{lo},{hi}): {m.sum()} rays, secant {sec[m].mean():.2f} us ({(sec[m] / np.maximum(it[m], 1)).mean():.3f} us/iter)")
    fin = np.sort(t1 - base) / 1e3
    print("  finished by (us) 50/90/99/100%:", [round(float(fin[int(q * (nb - 1))]), 1) for q in (0.5, 0.9, 0.99, 1.0)])
