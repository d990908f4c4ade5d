"""Per-ray timing of the ray-bounds kernel on the C4 bench sequence (debug aid).

Runs the bench's C4 frames through a graph-less tracker and, for frames >= FIRST, has the
library dump per-ray device start/end times and DDA step counts (SF_RB_DEBUG), then prints
the kernel span, the longest rays and the distribution of ray durations.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1311_7194_b200 as sf  # noqa: E402

FIRST = int(sys.argv[1]) if len(sys.argv) > 1 else 40
out = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/rb_debug.bin"
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
        os.environ["SF_RB_DEBUG"] = out
    if bench.reseed_due(c, k) and k > 0:
        tr.set_pose(poses[k - 1], stream=sp)
    tr.step(dframes[k], sf.Tracker.TRACK_WITH_HOOK, hooks[k], stream=sp)
    tr.fetch(stream=sp)
os.environ.pop("SF_RB_DEBUG", None)
n = c["width"] * c["height"]
d = np.fromfile(out, dtype=np.uint64).reshape(-1, n, 3)
for f in range(d.shape[0]):
    t0, t1, st = d[f, :, 0].astype(np.int64), d[f, :, 1].astype(np.int64), d[f, :, 2]
    steps = (st & 0xFFFF).astype(np.int64)
    jumps = ((st >> 16) & 0xFFFF).astype(np.int64)
    cta = (st >> 32).astype(np.int64)
    base = t0.min()
    dur = t1 - t0
    span = t1.max() - base
    print(f"frame {FIRST + f}: span {span / 1e3:.1f} us, rays {n}, steps total {steps.sum()}, max {steps.max()}")
    print("  ray duration us percentiles 50/90/99/99.9/max:",
          [round(float(np.percentile(dur, q)) / 1e3, 2) for q in (50, 90, 99, 99.9, 100)])
    print("  jumps percentiles 50/90/99/max:", [int(np.percentile(jumps, q)) for q in (50, 90, 99, 100)])
    for lo_, hi_ in ((0, 1), (1, 2), (2, 4), (4, 8), (8, 100)):
        m = (jumps >= lo_) & (jumps < hi_)
        if m.any():
            print(f"   jumps in [{lo_},{hi_}): {m.sum()} rays, mean dur {dur[m].mean() / 1e3:.1f} us, mean steps {steps[m].mean():.1f}")
    print("  steps percentiles 50/90/99/99.9/max:", [int(np.percentile(steps, q)) for q in (50, 90, 99, 99.9, 100)])
    order = np.argsort(-dur)[:8]
    for i in order:
        print(f"   px ({i % c['width']},{i // c['width']}) start {(t0[i] - base) / 1e3:.1f} dur {dur[i] / 1e3:.1f} us "
              f"steps {steps[i]} jumps {jumps[i]} cta {cta[i]}")
    # when do rays finish: fraction of rays finished at 50/75/90/100 % of the span
    fin = np.sort(t1 - base)
    print("  time by which 50/90/99/100% of rays finished (us):",
          [round(float(fin[int(q * (n - 1))]) / 1e3, 1) for q in (0.5, 0.9, 0.99, 1.0)])
    # per-CTA finish
    last = np.zeros(cta.max() + 1)
    np.maximum.at(last, cta, (t1 - base) / 1e3)
    print("  CTA finish times us percentiles 10/50/90/max:",
          [round(float(np.percentile(last, q)), 1) for q in (10, 50, 90, 100)])
