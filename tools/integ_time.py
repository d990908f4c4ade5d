"""Timing driver (not a test): the bench's integrate-only measurement (C4 frames at ground-truth
poses through the tracker, integrate kernel timed by its in-graph event pair, L2 flushed),
for the codes and float2 layouts. Prints ms per launch and the roofline fraction."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1311_7194_b200 as sfp
from paper_1311_7194_b200 import api as sf

steps, warm = 20, 5
c = bench.workload_config()
grid_cfg, intr, fusion, match = bench.make_params(sfp, c)
n = 1 + warm + steps
poses, frames = bench.make_frames(sfp, c, n, intr)
dev = torch.device("cuda", 0)
df = [sf.DepthFrame(intr, torch.from_numpy(f.depth).to(dev), torch.from_numpy(f.sigma).to(dev)) for f in frames]
flush = torch.empty(400 << 20, dtype=torch.uint8, device=dev)
sp = torch.cuda.current_stream().cuda_stream
peak = bench.hbm_peak()[0]
for name, lay, bpv in (("codes", sf.SparseTsdfGrid.CODES, 4), ("float2", sf.SparseTsdfGrid.FLOAT2, 16)):
    for rep in range(int(os.environ.get("REPS", "1"))):
        g = sf.SparseTsdfGrid(grid_cfg, c["pool"], sf.AuxMode.Variance, p_min=c["p_min"])
        g.set_payload_layout(lay)
        tr = sf.Tracker(g, intr, fusion, match, poses[0])
        tr.set_stage_timing(1)
        for k in range(1 + warm):
            tr.step(df[k], sf.Tracker.GROUND_TRUTH, poses[k], stream=sp)
        tr.fetch(stream=sp)
        ms, byt, ex, span = [], [], 0, []
        for i in range(steps):
            k = 1 + warm + i
            flush.fill_(i & 255)
            tr.step(df[k], sf.Tracker.GROUND_TRUTH, poses[k], stream=sp)
            m = tr.fetch(stream=sp)
            ms.append(tr.stage_times()[3])
            span.append(m.integrate_ns * 1e-6)
            byt.append(m.blocks_processed * (512 * bpv + 8) + 640 * 480 * 8)
            ex += m.exact_voxels
        t = sum(ms) / steps
        print(f"{name}: {t*1e3:.1f} us/launch (span {sum(span)/steps*1e3:.1f} us), frac {sum(byt)/(sum(ms)*1e-3)/1e9/peak:.3f}, "
              f"exact {ex/ (sum(b for b in byt))*0:.0f}{ex}")
