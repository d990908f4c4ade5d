"""Spatial sharding of the block pool across GPUs.

One process per GPU. Rank r's volume allocates only the blocks it owns
(owner = hash of the 8^3-block brick % world, ``sf_shard_owner``), so integration is split
with no data-path exchange: every voxel update depends only on its own prior and the frame
(fusion.cpp:294-366), and the union of the ranks' volumes equals the single volume bit for
bit. The per-frame loop of ``run()`` (pipeline.cpp:233-301) then needs three exchanges:

1. ray bounds: each rank runs the reference DDA over its own blocks; an all-reduce MIN of
   t_start and MAX of t_end gives exactly the single-volume bounds (the DDA visits the same
   cells with the same floating-point times on every rank, only occupancy differs);
2. halo: after integrating, each rank all-gathers the blocks it processed that touch another
   rank's brick, and mirrors (read-only) the ones touching its own bricks. Every sample the
   reference raycast takes around a crossing (bracket 0.5 delta apart, secant samples
   between, gradient +-1 voxel) is then evaluable on the rank owning the crossing's base voxel;
3. raycast: each rank marches its own and mirrored blocks from the global bounds. No rank
   can find an earlier crossing than the single volume (its valid samples are a subsequence
   of the global ones with the same values), and the owner of the true crossing finds it, so
   the nearest-depth composite — an all-reduce MIN of a per-pixel key (depth bits, normal
   flag, rank), then an all-reduce SUM of the winners' depth/normal bit patterns (int32; the
   losers contribute zeros, so the sum is a bit copy) — is the single-volume raycast;
4. ICP runs on the composited maps, identical on every rank (same inputs, deterministic
   kernels), and the fusion statistics are summed.

``LocalComm`` emulates R ranks inside one process (one GPU) with the same phase structure,
which is how the sharded path is parity-tested on a single B200; ``DistComm`` wraps
``torch.distributed`` (NCCL on device tensors, gloo on CPU tensors).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Optional

import torch

from . import _abi as A
from .api import (DepthFrame, FusionParams, FusionStats, Intrinsics, MatchParams, NormalMap, Pose,
                  RaycastStats, SparseTsdfGrid, _dptr, compose, default_backend, invert)

BRICK_SHIFT = 3  # owner granularity: 8^3 blocks


def shard_owner(bc, world: int, brick_shift: int = BRICK_SHIFT) -> int:
    """Owner rank of block coordinate ``bc`` (the device hash, sf_shard_owner)."""
    return int(default_backend().lib.shard_owner(int(bc[0]), int(bc[1]), int(bc[2]), brick_shift, world))


class LocalComm:
    """All ranks in this process: a collective reduces the per-rank tensors of one list."""

    def __init__(self, world: int):
        self.world = world
        self.ranks = list(range(world))

    def all_reduce(self, ts: List[torch.Tensor], op: str):
        assert len(ts) == self.world
        st = torch.stack(ts)
        if op == "min":
            r = st.amin(0)
        elif op == "max":
            r = st.amax(0)
        elif op == "sum":
            r = st.sum(0, dtype=st.dtype)
        else:
            raise ValueError(op)
        for t in ts:
            t.copy_(r)

    def exchange(self, recs):
        """recs[r] = (keys, payloads, count) of rank r -> for each rank, the other ranks' records."""
        return [[recs[q] for q in range(self.world) if q != r] for r in range(self.world)]


class DistComm:
    """This process is one rank of a torch.distributed group (NCCL for CUDA tensors)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.ranks = [dist.get_rank(group)]

    def all_reduce(self, ts: List[torch.Tensor], op: str):
        assert len(ts) == 1
        ops = {"min": self.dist.ReduceOp.MIN, "max": self.dist.ReduceOp.MAX, "sum": self.dist.ReduceOp.SUM}
        self.dist.all_reduce(ts[0], op=ops[op], group=self.group)

    def exchange(self, recs):
        """All-gather of variable-length halo records (padded to the largest count)."""
        keys, pays, count = recs[0]
        dev = keys.device
        cnt = torch.tensor([count], dtype=torch.int64, device=dev)
        counts = [torch.zeros_like(cnt) for _ in range(self.world)]
        self.dist.all_gather(counts, cnt, group=self.group)
        counts = [int(c.item()) for c in counts]
        mx = max(counts)
        if mx == 0:
            return [[]]
        if keys.shape[0] < mx:  # another rank packed more records than this rank's buffer holds
            keys = torch.cat([keys, keys.new_zeros(mx - keys.shape[0])])
            pays = torch.cat([pays, pays.new_zeros((mx - pays.shape[0],) + tuple(pays.shape[1:]))])
        k_send = keys[:mx].contiguous()
        p_send = pays[:mx].contiguous().view(torch.int32)  # NCCL / gloo have no 16-bit integer type
        k_all = [torch.empty_like(k_send) for _ in range(self.world)]
        p_all = [torch.empty_like(p_send) for _ in range(self.world)]
        self.dist.all_gather(k_all, k_send, group=self.group)
        self.dist.all_gather(p_all, p_send, group=self.group)
        me = self.ranks[0]
        return [[(k_all[q], p_all[q].view(torch.int16), counts[q]) for q in range(self.world) if q != me]]


class ShardVolume:
    """One rank's share of the block pool: a SparseTsdfGrid restricted to its own bricks."""

    def __init__(self, config, pool_capacity: int, aux_mode, rank: int, world: int,
                 brick_shift: int = BRICK_SHIFT, device: int = 0, **aux):
        self.rank, self.world = rank, world
        self.grid = SparseTsdfGrid(config, pool_capacity, aux_mode, device=device, **aux)
        be = self.grid.backend
        be.check(be.lib.volume_set_shard(self.grid.handle, rank, world, brick_shift))
        self.device = torch.device("cuda", device)

    def bounds(self, pose: Pose, intr: Intrinsics, ts: torch.Tensor, te: torch.Tensor):
        be = self.grid.backend
        ic = intr.c()
        be.check(be.lib.ray_bounds(self.grid.handle, _dptr(pose.to12()), C.byref(ic), ts.data_ptr(), te.data_ptr(),
                                   1, None))

    def march(self, pose: Pose, intr: Intrinsics, ts, te, depth, normals) -> RaycastStats:
        be = self.grid.backend
        ic = intr.c()
        st = A.RaycastStatsC()
        be.check(be.lib.raycast_with_bounds(self.grid.handle, _dptr(pose.to12()), C.byref(ic), ts.data_ptr(),
                                            te.data_ptr(), depth.data_ptr(), normals.data_ptr(), 1, C.byref(st),
                                            None))
        return RaycastStats(st.sample_steps, st.hit_pixels, st.rays_with_bounds)

    def fuse(self, frame: DepthFrame, pose: Pose, params: FusionParams) -> FusionStats:
        return self.grid.backend.fuse_frame(self.grid, frame, pose, params)

    def pack_halo(self):
        """(keys, payloads, count) of the last integrate's blocks bordering other ranks' bricks."""
        be = self.grid.backend
        m3 = self.grid.config.voxels_per_block_axis ** 3
        cap = getattr(self, "_cap", 0)
        cnt = C.c_uint32(0)
        while True:
            if cap == 0 or cap < getattr(self, "_need", 0):
                cap = max(4096, int(getattr(self, "_need", 0) * 1.25))
                self._keys = torch.empty(cap, dtype=torch.int32, device=self.device)
                self._pays = torch.empty((cap, m3), dtype=torch.int16, device=self.device)
                self._cap = cap
            st = be.lib.shard_pack_halo(self.grid.handle, self._keys.data_ptr(), self._pays.data_ptr(), cap,
                                        C.byref(cnt), None)
            if st == A.SF_OUT_OF_RANGE:
                self._need = cnt.value
                continue
            be.check(st)
            return self._keys, self._pays, cnt.value

    def apply_halo(self, keys, pays, count) -> int:
        be = self.grid.backend
        applied = C.c_uint32(0)
        be.check(be.lib.shard_apply_halo(self.grid.handle, keys.data_ptr(), pays.data_ptr(), count,
                                         C.byref(applied), None))
        return applied.value


def exchange_halo(shards: List[ShardVolume], comm):
    """After an integrate on every local rank: mirror the blocks bordering each rank's bricks."""
    if comm.world <= 1:
        return
    recs = [s.pack_halo() for s in shards]
    for s, incoming in zip(shards, comm.exchange(recs)):
        for keys, pays, count in incoming:
            if count:
                s.apply_halo(keys, pays, count)


def _composite(shards: List[ShardVolume], comm, depth: List[torch.Tensor], normals: List[torch.Tensor]):
    lib = default_backend().lib
    be = default_backend()
    n = depth[0].numel()
    keys = []
    for s, d, nm in zip(shards, depth, normals):
        k = torch.empty(n, dtype=torch.int64, device=d.device)
        be.check(lib.composite_key(d.data_ptr(), nm.data_ptr(), n, s.rank, k.data_ptr(), None))
        keys.append(k)
    comm.all_reduce(keys, "min")
    for s, k, d, nm in zip(shards, keys, depth, normals):
        be.check(lib.composite_select(k.data_ptr(), n, s.rank, d.data_ptr(), nm.data_ptr(), None))
    comm.all_reduce([d.view(torch.int32) for d in depth], "sum")
    comm.all_reduce([nm.view(torch.int32) for nm in normals], "sum")


def sharded_raycast(shards: List[ShardVolume], comm, pose: Pose, intr: Intrinsics):
    """raycast(grid, pose, intrinsics) over the union of the shards: global bounds, per-rank
    march, nearest-depth composite. Returns per local rank (depth (H,W), normals (H,W,3))
    device tensors, identical on every rank, and the summed per-rank stats."""
    h, w = intr.height, intr.width
    dev = shards[0].device
    ts = [torch.empty((h, w), dtype=torch.float32, device=dev) for _ in shards]
    te = [torch.empty((h, w), dtype=torch.float32, device=dev) for _ in shards]
    for s, a, b in zip(shards, ts, te):
        s.bounds(pose, intr, a, b)
    comm.all_reduce(ts, "min")
    comm.all_reduce(te, "max")
    depth = [torch.empty((h, w), dtype=torch.float32, device=dev) for _ in shards]
    normals = [torch.empty((h, w, 3), dtype=torch.float32, device=dev) for _ in shards]
    stats = [s.march(pose, intr, a, b, d, nm) for s, a, b, d, nm in zip(shards, ts, te, depth, normals)]
    _composite(shards, comm, depth, normals)
    return depth, normals, stats, ts, te


@dataclass
class ShardFrameMetrics:
    frame: int
    registered: bool
    pose: Pose
    iterations: int = 0
    matches: int = 0
    voxels_updated: int = 0  # summed over ranks
    blocks_total: int = 0    # summed over ranks
    hit_pixels: int = 0      # composite
    status: int = 0
    halo_records: int = 0    # native tracker: records packed this frame (all ranks)
    halo_overflow: int = 0   # records beyond the per-rank capacity (not exchanged)
    kernel_launches: int = 0
    icp_steps: int = 0


class ShardedTracker:
    """run() (pipeline.cpp:233-301) over a sharded block pool. ``shards`` are this process's
    ranks (one with DistComm, all with LocalComm)."""

    def __init__(self, shards: List[ShardVolume], comm, camera: Intrinsics, fusion: FusionParams,
                 match: MatchParams, initial_pose: Pose):
        self.shards, self.comm = shards, comm
        self.camera, self.fusion, self.match = camera, fusion, match
        self.current = initial_pose
        self.k = 0
        self.backend = default_backend()

    def step(self, captured: DepthFrame, external: Optional[Pose] = None, gt_pose: Optional[Pose] = None):
        """One frame. external: the icp_with_hook prior compose(invert(traj[k-1]), traj[k]);
        gt_pose: ground-truth tracking (no raycast / ICP)."""
        reg, it, nm_ = False, 0, 0
        hits = 0
        if self.k == 0:
            pose = self.current
        elif gt_pose is not None:
            pose = gt_pose
        else:
            depth, normals, _, _, _ = sharded_raycast(self.shards, self.comm, self.current, self.camera)
            hits = int((depth[0] > 0).sum().item())
            initial = compose(self.current, external) if external is not None else self.current
            initial_delta = compose(invert(self.current), initial)
            # identical inputs on every rank -> identical (deterministic) result; run once per process
            res = self.backend.icp(captured, DepthFrame(self.camera, depth[0]), NormalMap(normals[0]),
                                   initial_delta, self.match)
            pose = compose(self.current, res.delta)
            reg, it, nm_ = True, res.iterations, res.matches
        self.current = pose
        stats = [s.fuse(captured, pose, self.fusion) for s in self.shards]
        exchange_halo(self.shards, self.comm)
        dev = self.shards[0].device
        red = [torch.tensor([st.voxels_updated, st.blocks_total], dtype=torch.int64, device=dev) for st in stats]
        self.comm.all_reduce(red, "sum")
        vu, bt = (int(x) for x in red[0].tolist())
        m = ShardFrameMetrics(self.k, reg, pose, it, nm_, vu, bt, hits)
        self.k += 1
        return m


def broadcast_nccl_id(comm: "DistComm") -> bytes:
    """NCCL bootstrap of the native sharded frame: rank 0 makes the 128-byte ncclUniqueId
    (sf_nccl_unique_id) and the torch.distributed group broadcasts it to every rank."""
    import torch.distributed as dist

    obj = [None]
    if comm.ranks[0] == 0:
        uid = (C.c_uint8 * 128)()
        be = default_backend()
        be.check(be.lib.nccl_unique_id(uid))
        obj = [bytes(uid)]
    dist.broadcast_object_list(obj, src=0, group=comm.group)
    return obj[0]


class NativeShardedTracker:
    """The sharded fused frame as ONE CUDA graph per frame (sf_shard_tracker_*, csrc/sf_shard.cu):
    global ray bounds, per-rank march of the rays its own blocks meet, nearest-depth composite,
    ICP (``icp_mode`` 0: replicated; 1: partial sums over pixel slices + all-reduce), per-rank
    fuse and halo exchange, with no host synchronisation inside a frame. ``comm`` is a
    LocalComm (``shards`` = all ranks, in this process) or a DistComm (``shards`` = this rank;
    NCCL communicator bootstrapped through torch.distributed)."""

    TRACK, GROUND_TRUTH, TRACK_WITH_HOOK = 0, 1, 2

    def __init__(self, shards: List[ShardVolume], comm, camera: Intrinsics, fusion: FusionParams,
                 match: MatchParams, initial_pose: Pose, icp_mode: int = 0, halo_capacity: int = 0,
                 use_graphs: bool = True):
        self.shards, self.comm = shards, comm
        be = default_backend()
        self._lib = be.lib
        self.backend = be
        base = A.TrackerConfigC(fusion.c(), match.c(), camera.c(), 1 if use_graphs else 0, 0)
        cfg = A.ShardTrackerConfigC(base, int(icp_mode), 0, int(halo_capacity))
        p12 = initial_pose.to12()
        h = C.c_void_p()
        if isinstance(comm, DistComm):
            raw = (C.c_uint8 * 128).from_buffer_copy(broadcast_nccl_id(comm))
            be.check(self._lib.shard_tracker_create_nccl(shards[0].grid.handle, raw, comm.ranks[0], comm.world,
                                                         C.byref(cfg), _dptr(p12), C.byref(h)))
        else:
            vols = (C.c_void_p * len(shards))(*[s.grid.handle.value for s in shards])
            be.check(self._lib.shard_tracker_create_local(vols, len(shards), C.byref(cfg), _dptr(p12), C.byref(h)))
        self.handle = h

    def __del__(self):
        if getattr(self, "handle", None):
            try:
                self._lib.shard_tracker_destroy(self.handle)
            except Exception:
                pass
            self.handle = None

    def step(self, frame: DepthFrame, mode: int = 0, gt_pose: Optional[Pose] = None, stream=None):
        fc = frame.c()
        g = _dptr(gt_pose.to12()) if gt_pose is not None else None
        self.backend.check(self._lib.shard_tracker_step(self.handle, C.byref(fc), mode, g, stream))

    def set_pose(self, pose: Pose, stream=None):
        self.backend.check(self._lib.shard_tracker_set_pose(self.handle, _dptr(pose.to12()), stream))

    def fetch(self, stream=None) -> "ShardFrameMetrics":
        m = A.ShardFrameMetricsC()
        self.backend.check(self._lib.shard_tracker_fetch(self.handle, C.byref(m), stream))
        return ShardFrameMetrics(m.frame, bool(m.registered), Pose.from12(list(m.pose)), m.iterations, m.matches,
                                 m.voxels_updated, m.blocks_total, m.hit_pixels, m.status, m.halo_records,
                                 m.halo_overflow, m.kernel_launches, m.icp_steps)


def union_blocks(grids: List[SparseTsdfGrid], shards: Optional[List[ShardVolume]] = None):
    """{table index: payload block bytes} over the volumes (for parity checks); with ``shards``
    only each rank's own blocks (mirrored halo blocks excluded)."""
    out = {}
    for i, g in enumerate(grids):
        table = g.read_table()
        idx = (table >= 0).nonzero()[0]
        if shards is not None:
            n = g.config.blocks_per_axis
            s = shards[i]
            idx = [ti for ti in idx.tolist() if shard_owner((ti % n, (ti // n) % n, ti // (n * n)), s.world) == s.rank]
        if len(idx) == 0:
            continue
        pay = g.read_payload()
        m3 = g.config.voxels_per_block_axis ** 3
        for ti in list(idx):
            s = int(table[ti])
            if ti in out:
                raise AssertionError(f"block {ti} held by two shards")
            out[ti] = pay[s * m3:(s + 1) * m3].tobytes()
    return out
