import sys, os
sys.path.insert(0, '/root/repo')
import numpy as np
from paper_1311_7194_b200 import api as sf, shard
from tests import scenes
from tests.test_gpu_shard import _small_c5, _frames
gpu = sf.default_backend()
world = 2
intr = scenes.camera(320, 240, 262.5)
traj = scenes.c5_trajectory(100, radius=0.9)[:6]
cfg, _ = _small_c5(world)
frames = _frames(gpu, scenes.c5_scene(), traj, intr, cfg.box_side, sigma0=4e-4)
fusion = sf.FusionParams(mode=sf.FusionMode.Kalman)
match = sf.MatchParams.for_voxel_size(cfg.voxel_size)
cfg, sh1 = _small_c5(world)
tr = shard.NativeShardedTracker(sh1, shard.LocalComm(world), intr, fusion, match, traj[0])
cfg, sh2 = _small_c5(world)
tp = shard.ShardedTracker(sh2, shard.LocalComm(world), intr, fusion, match, traj[0])
for k, f in enumerate(frames):
    ext = sf.compose(sf.invert(traj[k - 1]), traj[k]) if k else sf.Pose.identity()
    tr.step(f, tr.TRACK_WITH_HOOK, ext); m = tr.fetch()
    mp = tp.step(f, external=ext if k else None)
    print(k, m.hit_pixels, mp.hit_pixels, m.matches, mp.matches, float(np.abs(m.pose.to12()-mp.pose.to12()).max()), m.halo_records)
