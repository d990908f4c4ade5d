"""GPU parity: the CUDA path against the oracle on identical inputs.

The oracle is the unmodified reference build (oracle/_ref) when present, else the C
restatement (oracle/liboracle.so, pinned bit-exact to the reference in
tests/test_oracle_cpu.py). Inputs are rendered by the product's GPU sphere tracer, which is
itself checked bit-exact against the reference. Bars (north star, BASELINE.json):
- integer / byte outputs (offset table, slots, payload codes, block lists): bit-exact;
- raycast depth / normals / ray bounds: bit-exact (FP64, reference operation order), which
  is stricter than the 1e-4-voxel bar;
- ICP pose: within 1e-6 (the 28 normal-equation sums are tree-reduced on the device).
"""
import ctypes as C
import math

import numpy as np
import pytest

from paper_1311_7194_b200 import api as sf
from tests import scenes

pytestmark = pytest.mark.gpu

POSE_TOL = 1e-6  # north star: ICP pose within 1e-6


def grids(gpu, ora, cfg, cap, aux_mode, **kw):
    return (sf.SparseTsdfGrid(cfg, cap, aux_mode, backend=gpu, **kw),
            sf.SparseTsdfGrid(cfg, cap, aux_mode, backend=ora, **kw))


def assert_same_volume(a, b):
    ta, tb = a.read_table(), b.read_table()
    assert np.array_equal(ta, tb), f"table differs at {np.flatnonzero(ta != tb)[:10]}"
    pa, pb = a.read_payload(), b.read_payload()
    diff = np.flatnonzero(pa != pb)
    assert diff.size == 0, f"{diff.size} payload codes differ, first {diff[:8]} gpu={pa[diff[:8]]} ref={pb[diff[:8]]}"
    assert a.allocated_count == b.allocated_count


def frames_for(gpu, scene, poses, intr, domain, sigma0=0.0):
    return [gpu.render_synthetic_depth(scene, p, intr, sigma0=sigma0, seed=1000 + k, domain_size=domain)
            for k, p in enumerate(poses)]


def pose_diff(a: sf.Pose, b: sf.Pose):
    return max(np.abs(a.rotation - b.rotation).max(), np.abs(a.translation - b.translation).max())


def pipeline_frame(be, grid, frame, intr, fusion, match, mode, ext, cur):
    """run()'s frame body (pipeline.cpp:250-287) over any backend's public API."""
    it = matches = 0
    if mode in (0, 2):
        d, n, _ = be.raycast(grid, cur, intr)
        init = sf.compose(cur, ext) if mode == 2 else cur  # initial_transform_hook
        res = be.icp(frame, d, n, sf.compose(sf.invert(cur), init), match)
        cur = sf.compose(cur, res.delta)
        it, matches = res.iterations, res.matches
    st = be.fuse_frame(grid, frame, cur, fusion)
    return cur, st, it, matches


# ---------------------------------------------------------------------------------
# input side
# ---------------------------------------------------------------------------------
@pytest.mark.parametrize("sigma0", [0.0, 2.5e-4])
def test_synthetic_depth_bit_exact(gpu, ref, sigma0):
    intr = scenes.camera(320, 240, 262.5)
    scene = scenes.sphere_plane_scene()
    scene.add_box([0.3, -0.2, 1.0], [0.1, 0.05, 0.08])
    pose = scenes.c1_trajectory(10)[3]
    a = gpu.render_synthetic_depth(scene, pose, intr, sigma0=sigma0, seed=77, domain_size=2.0)
    b = ref.render_synthetic_depth(scene, pose, intr, sigma0=sigma0, seed=77, domain_size=2.0)
    assert np.array_equal(a.depth, b.depth)
    if sigma0 > 0:
        assert np.array_equal(a.sigma, b.sigma)
    assert (a.depth > 0).mean() > 0.5


def test_synthetic_depth_vs_oracle(gpu, oracle):
    intr = scenes.camera(320, 240, 262.5)
    scene = scenes.bumpy_sphere()
    pose = scenes.c4_trajectory(10)[2]
    a = gpu.render_synthetic_depth(scene, pose, intr, domain_size=0.6144)
    b = oracle.render_synthetic_depth(scene, pose, intr, domain_size=0.6144)
    assert np.array_equal(a.depth, b.depth) and (a.depth > 0).sum() > 1000


@pytest.mark.parametrize("spatial", [0.0, 0.0078125])
def test_compute_normals_bit_exact(gpu, oracle, spatial):
    intr = scenes.camera(320, 240, 262.5)
    pose = scenes.c1_trajectory(10)[5]
    f = gpu.render_synthetic_depth(scenes.sphere_plane_scene(), pose, intr, sigma0=2.5e-4, seed=3, domain_size=2.0)
    a = gpu.compute_normals(f, 2.5e-4, spatial).array
    b = oracle.compute_normals(f, 2.5e-4, spatial).array
    assert np.array_equal(a, b)
    assert (np.abs(a).sum(-1) > 0).mean() > 0.3


# ---------------------------------------------------------------------------------
# fuse_frame
# ---------------------------------------------------------------------------------
@pytest.mark.parametrize("mode", [sf.FusionMode.Kalman, sf.FusionMode.Weighted, sf.FusionMode.Simple])
def test_fuse_sequence_bit_exact_c1(gpu, oracle, mode):
    """C1 (256^3, N=32, M=8): table, slots and every payload code equal after every frame."""
    intr = scenes.camera(320, 240, 262.5)
    poses = scenes.c1_trajectory(100)[::12]
    frames = frames_for(gpu, scenes.sphere_plane_scene(), poses, intr, 2.0)
    aux = sf.AuxMode.Variance if mode == sf.FusionMode.Kalman else sf.AuxMode.Weight
    g, r = grids(gpu, oracle, scenes.c1_config(), 0, aux)
    params = sf.FusionParams(mode=mode)
    for f, p in zip(frames, poses):
        sg = gpu.fuse_frame(g, f, p, params)
        sr = oracle.fuse_frame(r, f, p, params)
        assert sg == sr
        assert_same_volume(g, r)
    assert sr.blocks_total > 200 and sr.voxels_updated > 10000


def test_fuse_full_resolution_noisy_kalman(gpu, oracle):
    """640x480 noisy frames with a sigma plane, Kalman, edge down-weighting on."""
    intr = scenes.camera()
    poses = scenes.c1_trajectory(100)[::33]
    frames = frames_for(gpu, scenes.sphere_plane_scene(), poses, intr, 2.0, sigma0=2.5e-4)
    g, r = grids(gpu, oracle, scenes.c1_config(), 0, sf.AuxMode.Variance)
    params = sf.FusionParams(mode=sf.FusionMode.Kalman, sigma0=2.5e-4)
    for f, p in zip(frames, poses):
        assert gpu.fuse_frame(g, f, p, params) == oracle.fuse_frame(r, f, p, params)
        assert_same_volume(g, r)


def test_fuse_c4_scale_kalman(gpu, oracle):
    """C4 geometry (0.15 mm voxels, p_min 1e-12) on a block window around the object."""
    intr = scenes.camera(320, 240, 262.5)
    side = 128 * 8 * 0.15e-3
    cfg = sf.GridConfig(128, 8, (-side / 2, -side / 2, 0.35 - side / 2), side, 0.0)
    poses = scenes.c4_trajectory(100)[:3]
    frames = frames_for(gpu, scenes.bumpy_sphere(), poses, intr, side, sigma0=4e-4)
    g, r = grids(gpu, oracle, cfg, 60000, sf.AuxMode.Variance, p_min=1e-12)
    params = sf.FusionParams(mode=sf.FusionMode.Kalman, sigma0=4e-4)
    for f, p in zip(frames, poses):
        assert gpu.fuse_frame(g, f, p, params) == oracle.fuse_frame(r, f, p, params)
    assert_same_volume(g, r)


def test_fuse_m4_exact_500(gpu, oracle):
    """C2 geometry: N=125, M=4 (500^3), stride 2 sampling."""
    intr = scenes.camera(320, 240, 262.5)
    poses = scenes.c1_trajectory(100)[::40]
    frames = frames_for(gpu, scenes.sphere_plane_scene(), poses, intr, 2.0)
    g, r = grids(gpu, oracle, scenes.c2_config(), 200000, sf.AuxMode.Variance)
    params = sf.FusionParams(mode=sf.FusionMode.Kalman)
    for f, p in zip(frames, poses):
        assert gpu.fuse_frame(g, f, p, params) == oracle.fuse_frame(r, f, p, params)
        assert_same_volume(g, r)


def test_empty_and_ragged_frames(gpu, oracle):
    """Edge cases: an all-invalid frame, a 1-pixel-wide frame, an odd-sized frame."""
    p = scenes.c1_trajectory(10)[0]
    for w, h in [(64, 48), (1, 37), (97, 13)]:
        intr = sf.Intrinsics.simple(w, h, 60.0)
        g, r = grids(gpu, oracle, scenes.c1_config(), 0, sf.AuxMode.Weight)
        empty = sf.DepthFrame(intr, np.zeros((h, w), np.float32))
        assert gpu.fuse_frame(g, empty, p, sf.FusionParams()) == oracle.fuse_frame(r, empty, p, sf.FusionParams())
        f = gpu.render_synthetic_depth(scenes.sphere_plane_scene(), p, intr, domain_size=2.0)
        assert gpu.fuse_frame(g, f, p, sf.FusionParams()) == oracle.fuse_frame(r, f, p, sf.FusionParams())
        assert_same_volume(g, r)


def test_select_update_blocks_lists(gpu, oracle):
    intr = scenes.camera(320, 240, 262.5)
    poses = scenes.c1_trajectory(100)
    scene = scenes.sphere_plane_scene()
    g, r = grids(gpu, oracle, scenes.c1_config(), 0, sf.AuxMode.Weight)
    params = sf.FusionParams()
    for k in (0, 20, 40):
        f = gpu.render_synthetic_depth(scene, poses[k], intr, domain_size=2.0)
        ga, gu = gpu.select_update_blocks(g, f, poses[k])
        ra, ru = oracle.select_update_blocks(r, f, poses[k])
        assert np.array_equal(ga, ra)
        assert np.array_equal(gu, ru)
        gpu.fuse_frame(g, f, poses[k], params)
        oracle.fuse_frame(r, f, poses[k], params)
    assert len(ru) > 0


def test_float_payload_matches_reference_shadow(gpu, ref):
    """Float payload mode == FloatShadowGrid semantics (grid.hpp:77-88, fusion.cpp:313-318)."""
    cfg = sf.GridConfig(16, 8, (-1.0, -1.0, 0.25), 2.0, 0.0)  # 128^3: shadow limit
    intr = scenes.camera(320, 240, 262.5)
    poses = scenes.c1_trajectory(100)[::25]
    frames = frames_for(gpu, scenes.sphere_plane_scene(), poses, intr, 2.0, sigma0=2.5e-4)
    g, r = grids(gpu, ref, cfg, 4096, sf.AuxMode.Variance)
    g.enable_float_payload()
    assert ref.lib.volume_enable_shadow(r.handle) == 0
    params = sf.FusionParams(mode=sf.FusionMode.Kalman)
    for f, p in zip(frames, poses):
        assert gpu.fuse_frame(g, f, p, params) == ref.fuse_frame(r, f, p, params)
    assert_same_volume(g, r)
    res = 128
    st = np.zeros(res ** 3, np.float32)
    sa = np.zeros(res ** 3, np.float32)
    ref.lib.volume_read_shadow(r.handle, st.ctypes.data_as(C.POINTER(C.c_float)),
                               sa.ctypes.data_as(C.POINTER(C.c_float)))
    fp = g.read_float_payload()
    table = g.read_table()
    n, m = 16, 8
    compared = 0
    for ti in np.flatnonzero(table >= 0):
        slot = table[ti]
        bx, by, bz = ti % n, (ti // n) % n, ti // (n * n)
        blk = fp[slot * 512:(slot + 1) * 512].reshape(m, m, m, 2)  # z, y, x
        dense_t = st.reshape(res, res, res)[bz * m:(bz + 1) * m, by * m:(by + 1) * m, bx * m:(bx + 1) * m]
        dense_a = sa.reshape(res, res, res)[bz * m:(bz + 1) * m, by * m:(by + 1) * m, bx * m:(bx + 1) * m]
        assert np.array_equal(blk[..., 0], dense_t)
        assert np.array_equal(blk[..., 1], dense_a)
        compared += 1
    assert compared > 50


def _assert_float_close(a, b, what):
    """Float payload bar (north star): chi pattern equal; TSDF within 1e-5 absolute; aux
    (variance / weight) within 1e-5 relative."""
    chi_a, chi_b = ~(a[:, 0] < np.inf), ~(b[:, 0] < np.inf)
    assert np.array_equal(chi_a, chi_b), f"{what}: chi pattern differs at {np.flatnonzero(chi_a != chi_b)[:8]}"
    live = ~chi_a
    assert np.abs(a[live, 0].astype(np.float64) - b[live, 0]).max(initial=0) <= 1e-5, what
    rel = np.abs(a[live, 1].astype(np.float64) - b[live, 1]) / np.maximum(np.abs(b[live, 1]), 1e-300)
    assert rel.max(initial=0) <= 1e-5, f"{what}: aux rel diff {rel.max()}"
    assert np.all(a[chi_a, 1] == 0)
    return int(live.sum())


@pytest.mark.parametrize("mode", [sf.FusionMode.Kalman, sf.FusionMode.Weighted, sf.FusionMode.Simple])
def test_float2_payload_matches_reference_shadow(gpu, ref, mode):
    """SF_PAYLOAD_FLOAT2 (P2: float {tsdf, aux} only, the FP32 row kernel with certified
    decisions) against the reference's FloatShadowGrid (grid.hpp:77-88, fusion.cpp:313-318,
    357-361): offset table bit-exact, chi pattern equal, values within 1e-5."""
    cfg = sf.GridConfig(16, 8, (-1.0, -1.0, 0.25), 2.0, 0.0)  # 128^3: the reference shadow's limit
    intr = scenes.camera(320, 240, 262.5)
    poses = scenes.c1_trajectory(100)[::25]
    frames = frames_for(gpu, scenes.sphere_plane_scene(), poses, intr, 2.0, sigma0=2.5e-4)
    aux = sf.AuxMode.Variance if mode == sf.FusionMode.Kalman else sf.AuxMode.Weight
    g, r = grids(gpu, ref, cfg, 4096, aux)
    g.set_payload_layout(g.FLOAT2)
    assert g.payload_layout == g.FLOAT2
    assert ref.lib.volume_enable_shadow(r.handle) == 0
    params = sf.FusionParams(mode=mode, sigma0=2.5e-4)
    for f, p in zip(frames, poses):
        assert gpu.fuse_frame(g, f, p, params) == ref.fuse_frame(r, f, p, params)
    assert np.array_equal(g.read_table(), r.read_table())
    res, n, m = 128, 16, 8
    st = np.zeros(res ** 3, np.float32)
    sa = np.zeros(res ** 3, np.float32)
    ref.lib.volume_read_shadow(r.handle, st.ctypes.data_as(C.POINTER(C.c_float)),
                               sa.ctypes.data_as(C.POINTER(C.c_float)))
    fp = g.read_float_payload()
    table = g.read_table()
    ours, theirs = [], []
    for ti in np.flatnonzero(table >= 0):
        slot = table[ti]
        bx, by, bz = ti % n, (ti // n) % n, ti // (n * n)
        ours.append(fp[slot * 512:(slot + 1) * 512])
        dt = st.reshape(res, res, res)[bz * m:(bz + 1) * m, by * m:(by + 1) * m, bx * m:(bx + 1) * m].reshape(-1)
        da = sa.reshape(res, res, res)[bz * m:(bz + 1) * m, by * m:(by + 1) * m, bx * m:(bx + 1) * m].reshape(-1)
        theirs.append(np.stack([dt, da], -1))
    live = _assert_float_close(np.concatenate(ours), np.concatenate(theirs), "float2 vs shadow")
    assert live > 20000
    with pytest.raises(NotImplementedError):
        gpu.raycast(g, poses[-1], intr)  # codes are not maintained on a float2 volume


def test_float2_payload_c4_scale(gpu, workload_c4):
    """P2 at the benchmarked C4 geometry (N = 512, 640x480 noisy frames, Kalman, p_min 1e-12):
    the float2 row kernel against the FP64 float-shadow kernel (itself equal to the reference's
    FloatShadowGrid above): same blocks, chi pattern, values within 1e-5."""
    c, grid_cfg, intr, fusion, poses, frames = workload_c4
    a = sf.SparseTsdfGrid(grid_cfg, c["pool"], sf.AuxMode.Variance, p_min=c["p_min"], backend=gpu)
    b = sf.SparseTsdfGrid(grid_cfg, c["pool"], sf.AuxMode.Variance, p_min=c["p_min"], backend=gpu)
    a.set_payload_layout(a.FLOAT2)
    b.enable_float_payload()
    for f, p in zip(frames, poses):
        assert gpu.fuse_frame(a, f, p, fusion) == gpu.fuse_frame(b, f, p, fusion)
    assert np.array_equal(a.read_table(), b.read_table())
    n = b.allocated_count
    live = _assert_float_close(a.read_float_payload(0, n), b.read_float_payload(0, n), "float2 C4")
    assert live > 1_000_000


def _axis_poses():
    """Cameras whose optical axes are closest to x, y and z in turn, so the integrate kernel's
    rows (along the block axis with the largest camera-z component) run along each axis: the
    half-block slab layouts of all three row axes are exercised."""
    import math
    around_x = sf.orbit_trajectory([0.0, 0.0, 1.3], 1.3, 4, (1.0, 0.0, 0.0), 0.05, math.pi / 2)  # +y .. +z
    around_y = sf.orbit_trajectory([0.0, 0.0, 1.3], 1.3, 2, (0.0, 1.0, 0.0), 0.1, 0.4)  # -x
    poses = around_x + around_y
    axes = {int(np.argmax(np.abs(p.rotation[:, 2]))) for p in poses}  # world axis of the camera's z
    assert axes == {0, 1, 2}, axes
    return poses


@pytest.mark.parametrize("mode", [sf.FusionMode.Kalman, sf.FusionMode.Weighted, sf.FusionMode.Simple])
def test_fuse_all_row_axes_bit_exact(gpu, oracle, mode):
    """Codes layout, every row axis of the slab kernel: stats, table and payload bit-exact."""
    intr = scenes.camera(320, 240, 262.5)
    poses = _axis_poses()
    frames = frames_for(gpu, scenes.sphere_plane_scene(), poses, intr, 2.0, sigma0=2.5e-4)
    aux = sf.AuxMode.Variance if mode == sf.FusionMode.Kalman else sf.AuxMode.Weight
    g, r = grids(gpu, oracle, scenes.c1_config(), 20000, aux)
    params = sf.FusionParams(mode=mode, sigma0=2.5e-4)
    for f, p in zip(frames, poses):
        assert gpu.fuse_frame(g, f, p, params) == oracle.fuse_frame(r, f, p, params)
        assert_same_volume(g, r)


def test_float2_all_row_axes_match_reference_shadow(gpu, ref):
    """Float2 layout, every row axis of the slab kernel, against the reference's FloatShadowGrid."""
    cfg = sf.GridConfig(16, 8, (-1.0, -1.0, 0.25), 2.0, 0.0)  # 128^3: the reference shadow's limit
    intr = scenes.camera(320, 240, 262.5)
    poses = _axis_poses()
    frames = frames_for(gpu, scenes.sphere_plane_scene(), poses, intr, 2.0, sigma0=2.5e-4)
    g, r = grids(gpu, ref, cfg, 4096, sf.AuxMode.Variance)
    g.set_payload_layout(g.FLOAT2)
    assert ref.lib.volume_enable_shadow(r.handle) == 0
    params = sf.FusionParams(mode=sf.FusionMode.Kalman, sigma0=2.5e-4)
    for f, p in zip(frames, poses):
        assert gpu.fuse_frame(g, f, p, params) == ref.fuse_frame(r, f, p, params)
    assert np.array_equal(g.read_table(), r.read_table())
    res, n, m = 128, 16, 8
    st = np.zeros(res ** 3, np.float32)
    sa = np.zeros(res ** 3, np.float32)
    ref.lib.volume_read_shadow(r.handle, st.ctypes.data_as(C.POINTER(C.c_float)),
                               sa.ctypes.data_as(C.POINTER(C.c_float)))
    fp = g.read_float_payload()
    table = g.read_table()
    ours, theirs = [], []
    for ti in np.flatnonzero(table >= 0):
        slot = table[ti]
        bx, by, bz = ti % n, (ti // n) % n, ti // (n * n)
        ours.append(fp[slot * 512:(slot + 1) * 512])
        dt = st.reshape(res, res, res)[bz * m:(bz + 1) * m, by * m:(by + 1) * m, bx * m:(bx + 1) * m].reshape(-1)
        da = sa.reshape(res, res, res)[bz * m:(bz + 1) * m, by * m:(by + 1) * m, bx * m:(bx + 1) * m].reshape(-1)
        theirs.append(np.stack([dt, da], -1))
    live = _assert_float_close(np.concatenate(ours), np.concatenate(theirs), "float2 vs shadow, all axes")
    assert live > 10000


@pytest.fixture(scope="module")
def workload_c4(gpu):
    import bench
    import paper_1311_7194_b200 as sfp

    c = bench.workload_config()
    grid_cfg, intr, fusion, _ = bench.make_params(sfp, c)
    poses, frames = bench.make_frames(sfp, c, 4, intr)
    return c, grid_cfg, intr, fusion, poses, frames


def test_pool_exhaustion_partial_state(gpu, oracle):
    """PoolExhausted mid-list: the allocate-list prefix is integrated, nothing else (fusion.cpp:369)."""
    intr = scenes.camera(320, 240, 262.5)
    pose = scenes.c1_trajectory(100)[10]
    f = gpu.render_synthetic_depth(scenes.sphere_plane_scene(), pose, intr, domain_size=2.0)
    g, r = grids(gpu, oracle, scenes.c1_config(), 150, sf.AuxMode.Weight)
    params = sf.FusionParams()
    with pytest.raises(sf.PoolExhausted):
        oracle.fuse_frame(r, f, pose, params)
    with pytest.raises(sf.PoolExhausted):
        gpu.fuse_frame(g, f, pose, params)
    assert r.allocated_count == 150
    assert_same_volume(g, r)


def test_grid_api_parity(gpu, oracle):
    cfg = sf.GridConfig(8, 4, (0, 0, 0), 1.0, 0.0)
    g, r = grids(gpu, oracle, cfg, 20, sf.AuxMode.Weight)
    rng = np.random.default_rng(5)
    for _ in range(300):
        bc = rng.integers(0, 8, 3)
        op = rng.integers(0, 3)
        if op == 0:
            try:
                a = r.allocate_block(bc)
            except sf.PoolExhausted:
                with pytest.raises(sf.PoolExhausted):
                    g.allocate_block(bc)
                continue
            assert g.allocate_block(bc) == a
        elif op == 1:
            r.free_block(bc)
            g.free_block(bc)
        else:
            vc = bc * 4 + rng.integers(0, 4, 3)
            t = float(rng.uniform(-0.6, 0.6)) * r.delta
            aux = float(rng.uniform(0, 25))
            try:
                r.write_voxel(vc, t, aux)
            except RuntimeError:
                with pytest.raises(RuntimeError):
                    g.write_voxel(vc, t, aux)
                continue
            g.write_voxel(vc, t, aux)
            assert g.read_voxel(vc) == r.read_voxel(vc)
    assert_same_volume(g, r)
    with pytest.raises(IndexError):
        g.allocate_block([8, 0, 0])


def test_snapshot_roundtrip_cross_implementation(gpu, ref, tmp_path):
    intr = scenes.camera(320, 240, 262.5)
    pose = scenes.c1_trajectory(100)[30]
    f = gpu.render_synthetic_depth(scenes.sphere_plane_scene(), pose, intr, domain_size=2.0)
    g, r = grids(gpu, ref, scenes.c1_config(), 0, sf.AuxMode.Weight)
    gpu.fuse_frame(g, f, pose, sf.FusionParams())
    ref.fuse_frame(r, f, pose, sf.FusionParams())
    pg, pr = str(tmp_path / "g.stsg"), str(tmp_path / "r.stsg")
    g.save_snapshot(pg)
    r.save_snapshot(pr)
    assert open(pg, "rb").read() == open(pr, "rb").read()
    g2 = sf.SparseTsdfGrid.load_snapshot(pr, backend=gpu)
    r2 = sf.SparseTsdfGrid.load_snapshot(pr, backend=ref)
    assert_same_volume(g2, r2)


def test_dfrm_device_buffers(gpu, ref, tmp_path):
    """DFRM (frame_io.cpp:28-79) from and into DEVICE buffers: writing a device-resident frame
    gives the reference's bytes; reading into device buffers gives the host read's planes, and
    fusing straight from them equals fusing the host frame."""
    import torch

    intr = scenes.camera(320, 240, 262.5)
    pose = scenes.c1_trajectory(100)[20]
    f = gpu.render_synthetic_depth(scenes.sphere_plane_scene(), pose, intr, sigma0=2.5e-4, seed=4, domain_size=2.0)
    dev = torch.device("cuda", 0)
    fd = sf.DepthFrame(intr, torch.from_numpy(f.depth).to(dev), torch.from_numpy(f.sigma).to(dev))
    a, b = str(tmp_path / "dev.dfrm"), str(tmp_path / "ref.dfrm")
    gpu.write_dfrm(fd, a)
    ref.write_dfrm(f, b)
    assert open(a, "rb").read() == open(b, "rb").read()
    rd = gpu.read_dfrm(b, device=dev)
    rh = ref.read_dfrm(b)
    assert rd.depth.is_cuda and rd.sigma is not None
    assert np.array_equal(rd.depth.cpu().numpy(), rh.depth) and np.array_equal(rd.sigma.cpu().numpy(), rh.sigma)
    g1, r = grids(gpu, ref, scenes.c1_config(), 0, sf.AuxMode.Variance)
    g2 = sf.SparseTsdfGrid(scenes.c1_config(), 0, sf.AuxMode.Variance, backend=gpu)
    params = sf.FusionParams(mode=sf.FusionMode.Kalman, sigma0=2.5e-4)
    assert gpu.fuse_frame(g1, rd, pose, params) == gpu.fuse_frame(g2, rh, pose, params) == ref.fuse_frame(r, rh, pose, params)
    assert_same_volume(g1, r)
    assert_same_volume(g2, r)


def test_snapshot_resume_on_device(gpu, ref, tmp_path):
    """Resume from an STSG snapshot (grid.cpp:333-408): the reference fuses and saves, the device
    volume loads it and both keep fusing; volumes and re-saved snapshots stay identical."""
    intr = scenes.camera(320, 240, 262.5)
    poses = scenes.c1_trajectory(100)[10:50:10]
    frames = frames_for(gpu, scenes.sphere_plane_scene(), poses, intr, 2.0, sigma0=2.5e-4)
    params = sf.FusionParams(mode=sf.FusionMode.Kalman, sigma0=2.5e-4)
    r = sf.SparseTsdfGrid(scenes.c1_config(), 3000, sf.AuxMode.Variance, backend=ref)
    for f, p in zip(frames[:2], poses[:2]):
        ref.fuse_frame(r, f, p, params)
    path = str(tmp_path / "mid.stsg")
    r.save_snapshot(path)
    g = sf.SparseTsdfGrid.load_snapshot(path, pool_capacity=3000, backend=gpu)
    assert_same_volume(g, r)
    for f, p in zip(frames[2:], poses[2:]):
        assert gpu.fuse_frame(g, f, p, params) == ref.fuse_frame(r, f, p, params)
    assert_same_volume(g, r)
    pg, pr = str(tmp_path / "g.stsg"), str(tmp_path / "r.stsg")
    g.save_snapshot(pg)
    r.save_snapshot(pr)
    assert open(pg, "rb").read() == open(pr, "rb").read()


# ---------------------------------------------------------------------------------
# raycast
# ---------------------------------------------------------------------------------
def fused_pair(gpu, ora, cfg, intr, poses, scene, domain, mode=sf.FusionMode.Weighted, cap=0, **kw):
    aux = sf.AuxMode.Variance if mode == sf.FusionMode.Kalman else sf.AuxMode.Weight
    g, r = grids(gpu, ora, cfg, cap, aux, **kw)
    params = sf.FusionParams(mode=mode)
    for p in poses:
        f = gpu.render_synthetic_depth(scene, p, intr, domain_size=domain)
        gpu.fuse_frame(g, f, p, params)
        ora.fuse_frame(r, f, p, params)
    assert_same_volume(g, r)
    return g, r


def check_raycast(gpu, ora, g, r, pose, intr, min_hits):
    gs, ge = gpu.compute_ray_bounds(g, pose, intr)
    rs, re_ = ora.compute_ray_bounds(r, pose, intr)
    assert np.array_equal(gs, rs) and np.array_equal(ge, re_)
    gd, gn, gst = gpu.raycast_result(g, pose, intr)
    rd, rn, rst = ora.raycast_result(r, pose, intr)
    assert gst == rst
    assert np.array_equal(gd.depth, rd.depth)
    assert np.array_equal(gn.array, rn.array)
    assert rst.hit_pixels > min_hits


def test_ray_bounds_and_raycast_bit_exact(gpu, oracle):
    intr = scenes.camera(320, 240, 262.5)
    poses = scenes.c1_trajectory(100)
    g, r = fused_pair(gpu, oracle, scenes.c1_config(), intr, poses[::20], scenes.sphere_plane_scene(), 2.0)
    for p in (poses[10], poses[55]):
        check_raycast(gpu, oracle, g, r, p, intr, 10000)
    # a camera inside the volume box, close to the surface
    inside = sf.Pose(poses[40].rotation, np.array([0.0, 0.0, 0.5]))
    check_raycast(gpu, oracle, g, r, inside, intr, 100)


def test_raycast_m4_kalman(gpu, oracle):
    intr = scenes.camera(320, 240, 262.5)
    poses = scenes.c1_trajectory(100)
    g, r = fused_pair(gpu, oracle, scenes.c2_config(), intr, poses[::30], scenes.sphere_plane_scene(), 2.0,
                      sf.FusionMode.Kalman, cap=200000)
    check_raycast(gpu, oracle, g, r, poses[45], intr, 10000)


def test_raycast_c4_scale(gpu, oracle):
    intr = scenes.camera(320, 240, 262.5)
    side = 128 * 8 * 0.15e-3
    cfg = sf.GridConfig(128, 8, (-side / 2, -side / 2, 0.35 - side / 2), side, 0.0)
    poses = scenes.c4_trajectory(100)
    g, r = fused_pair(gpu, oracle, cfg, intr, poses[:3], scenes.bumpy_sphere(), side, cap=60000)
    check_raycast(gpu, oracle, g, r, poses[3], intr, 500)


def test_raycast_empty_volume(gpu, oracle):
    intr = scenes.camera(64, 48, 55.0)
    g, r = grids(gpu, oracle, scenes.c1_config(), 0, sf.AuxMode.Weight)
    check_raycast(gpu, oracle, g, r, scenes.c1_trajectory(10)[0], intr, -1)


# ---------------------------------------------------------------------------------
# ICP
# ---------------------------------------------------------------------------------
def test_icp_recovers_perturbation_like_reference(gpu, oracle):
    """test_smoke.py:102-130 scenario at 320x240."""
    intr = scenes.camera(320, 240, 280.0)
    scene = scenes.cluster_scene()
    target_pose = sf.orbit_trajectory([0.0, 0.0, 1.3], 1.3, 8)[1]
    ang = math.radians(2.0)
    perturb = sf.Pose([[math.cos(ang), 0, math.sin(ang)], [0, 1, 0], [-math.sin(ang), 0, math.cos(ang)]],
                      [0.01, -0.005, 0.008])
    source_pose = sf.compose(target_pose, perturb)
    target = gpu.render_synthetic_depth(scene, target_pose, intr)
    source = gpu.render_synthetic_depth(scene, source_pose, intr)
    tn = gpu.compute_normals(target, 2.5e-4, 0.006)
    params = sf.MatchParams.for_voxel_size(1.5 / 256.0)
    a = gpu.icp(source, target, tn, sf.Pose.identity(), params)
    b = oracle.icp(source, target, tn, sf.Pose.identity(), params)
    assert a.iterations == b.iterations
    assert a.matches == b.matches
    assert pose_diff(a.delta, b.delta) < POSE_TOL
    assert a.gated_mask == b.gated_mask
    np.testing.assert_allclose(a.eigenvalues, b.eigenvalues, rtol=1e-9)
    truth = sf.compose(sf.invert(target_pose), source_pose)
    assert pose_diff(a.delta, truth) < 1e-3


def test_icp_against_raycast_model(gpu, oracle):
    """ICP of a captured frame against the raycast model, as run() does."""
    intr = scenes.camera(320, 240, 262.5)
    poses = scenes.c1_trajectory(100)
    g, r = fused_pair(gpu, oracle, scenes.c1_config(), intr, poses[:40:4], scenes.sphere_plane_scene(), 2.0)
    cur = poses[40]
    rd, rn, _ = oracle.raycast(r, cur, intr)
    captured = gpu.render_synthetic_depth(scenes.sphere_plane_scene(), poses[41], intr, domain_size=2.0)
    params = sf.MatchParams.for_voxel_size(2.0 / 256)
    init = sf.compose(sf.invert(cur), cur)
    a = gpu.icp(captured, rd, rn, init, params)
    b = oracle.icp(captured, rd, rn, init, params)
    assert a.iterations == b.iterations and abs(int(a.matches) - int(b.matches)) <= 2
    assert pose_diff(a.delta, b.delta) < POSE_TOL


def test_icp_reference_order_bit_identical(gpu, ref):
    """MatchParams.reduction = REFERENCE_ORDER: the same delta pose, eigenpairs, gated mask,
    residual and counts as the reference's icp(), bit for bit (sequential Kahan sums in match
    order, cyclic Jacobi, spectral gated solve, SVD apply_motion)."""
    intr = scenes.camera(320, 240, 262.5)
    poses = scenes.c1_trajectory(100)[:12:3]
    cfg = scenes.c1_config()
    g, r = fused_pair(gpu, ref, cfg, intr, poses[:3], scenes.sphere_plane_scene(), 2.0)
    src = gpu.render_synthetic_depth(scenes.sphere_plane_scene(), poses[3], intr, sigma0=2.5e-4, seed=9,
                                     domain_size=2.0)
    d, n, _ = ref.raycast(r, poses[2], intr)
    match = sf.MatchParams.for_voxel_size(cfg.voxel_size)
    match.reduction = sf.MatchParams.REFERENCE_ORDER
    for init in (sf.Pose.identity(), sf.compose(sf.invert(poses[2]), poses[3])):
        a = gpu.icp(src, d, n, init, match)
        b = ref.icp(src, d, n, init, match)
        assert a.iterations == b.iterations and a.matches == b.matches and a.iterations >= 2
        assert np.array_equal(a.delta.to12(), b.delta.to12())
        assert a.residual_rms == b.residual_rms and a.shrunk_motion_norm == b.shrunk_motion_norm
        assert a.eigenvalues == b.eigenvalues and a.gated_mask == b.gated_mask
        assert np.array_equal(a.eigenvectors, b.eigenvectors)
        assert np.array_equal(a.motion_r, b.motion_r) and np.array_equal(a.motion_t, b.motion_t)


def test_icp_tracking_lost(gpu, oracle):
    intr = scenes.camera(64, 48, 55.0)
    empty = sf.DepthFrame(intr, np.zeros((48, 64), np.float32))
    nm = sf.NormalMap(np.zeros((48, 64, 3), np.float32))
    with pytest.raises(sf.TrackingLost):
        oracle.icp(empty, empty, nm, sf.Pose.identity(), sf.MatchParams())
    with pytest.raises(sf.TrackingLost):
        gpu.icp(empty, empty, nm, sf.Pose.identity(), sf.MatchParams())


# ---------------------------------------------------------------------------------
# fused frame loop (run() body)
# ---------------------------------------------------------------------------------
@pytest.mark.parametrize("hook", [False, True])
def test_tracker_matches_reference_pipeline(gpu, oracle, hook):
    """C2-style full loop (raycast -> ICP -> fuse, tracking.mode icp / icp_with_hook) over a
    short sequence, with a relocalisation (set_pose) mid-way: poses within 1e-6, tables
    equal, payload codes equal up to the rare rounding-boundary voxel."""
    intr = scenes.camera(320, 240, 262.5)
    poses = scenes.c1_trajectory(100)[:10]
    frames = frames_for(gpu, scenes.sphere_plane_scene(), poses, intr, 2.0, sigma0=2.5e-4)
    cfg = scenes.c1_config()
    fusion = sf.FusionParams(mode=sf.FusionMode.Kalman, sigma0=2.5e-4)
    match = sf.MatchParams.for_voxel_size(cfg.voxel_size)
    g, r = grids(gpu, oracle, cfg, 0, sf.AuxMode.Variance)
    tr = sf.Tracker(g, intr, fusion, match, poses[0])
    cur = poses[0]
    mode = sf.Tracker.TRACK_WITH_HOOK if hook else sf.Tracker.TRACK
    for k, f in enumerate(frames):
        ext = sf.compose(sf.invert(poses[k - 1]), poses[k]) if k else sf.Pose.identity()
        if k == 6:
            tr.set_pose(poses[5])
            cur = poses[5]
        tr.step(f, mode, ext if hook else None)
        m = tr.fetch()
        cur, st, it, matches = pipeline_frame(oracle, r, f, intr, fusion, match, mode if k else 1, ext, cur)
        assert m.status == 0
        assert pose_diff(m.pose, cur) < POSE_TOL
        if k > 0:
            # tree-ordered vs sequential-Kahan ICP sums differ by ~1 ulp: a projective
            # association sitting on a rounding boundary may flip for a pixel
            assert m.registered and m.iterations == it
            assert abs(int(m.matches) - int(matches)) <= max(8, matches // 2000)
        assert m.fusion.blocks_total == st.blocks_total
    assert np.array_equal(g.read_table(), r.read_table())
    assert (g.read_payload() == r.read_payload()).mean() > 0.9999
    assert tr.last_launch_count() > 10
    assert tr.fetch().kernel_launches > tr.last_launch_count()  # + the device-side ICP iterations


def reference_run(oracle, r, frames, intr, fusion, match, pose0):
    """run()'s loop incl. its catch blocks (pipeline.cpp:233-301) over the oracle: the
    FrameMetrics it pushes, as (status, registered, pose, fusion stats, iterations)."""
    cur, out = pose0, []
    for k, f in enumerate(frames):
        fm = dict(status=0, registered=False, pose=sf.Pose.identity(), fusion=sf.FusionStats(0, 0, 0, 0), it=0)
        try:
            if k == 0:
                fm["pose"] = cur
            else:
                d, n, _ = oracle.raycast(r, cur, intr)
                res = oracle.icp(f, d, n, sf.compose(sf.invert(cur), cur), match)
                fm.update(registered=True, it=res.iterations)
                cur = sf.compose(cur, res.delta)
                fm["pose"] = cur
            fm["fusion"] = oracle.fuse_frame(r, f, fm["pose"], fusion)
        except sf.TrackingLost:
            fm["status"] = 5
            out.append(fm)
            break
        except sf.PoolExhausted:
            fm["status"] = 4
            out.append(fm)
            break
        out.append(fm)
    return out


@pytest.mark.parametrize("failure", ["tracking_lost", "pool_exhausted"])
def test_tracker_failure_frame_matches_reference_run(gpu, oracle, failure):
    """The frame that raises TrackingLost / PoolExhausted reports what run()'s catch block
    pushes (pipeline.cpp:289-299): TrackingLost -> not registered, identity pose, default
    FusionStats; PoolExhausted -> the registration and pose, default FusionStats; the volume is
    the reference's partial state; later steps are no-ops with the same status."""
    intr = scenes.camera(160, 120, 131.25)
    poses = scenes.c1_trajectory(100)[:5]
    frames = [gpu.render_synthetic_depth(scenes.sphere_plane_scene(), p, intr, domain_size=2.0) for p in poses]
    cfg = scenes.c1_config()
    fusion = sf.FusionParams(mode=sf.FusionMode.Kalman)
    match = sf.MatchParams.for_voxel_size(cfg.voxel_size)
    cap = 0
    if failure == "tracking_lost":
        frames[3] = sf.DepthFrame(intr, np.zeros((120, 160), np.float32))  # < 10 matches
    else:
        # a pool that holds frames 0..k-1 and half of frame k's new blocks (k >= 2)
        _, r0 = grids(gpu, oracle, cfg, 0, sf.AuxMode.Variance)
        tot = [fm["fusion"].blocks_total for fm in reference_run(oracle, r0, frames, intr, fusion, match, poses[0])]
        k = next(k for k in range(2, len(tot)) if tot[k] - tot[k - 1] >= 2)
        cap = tot[k - 1] + (tot[k] - tot[k - 1]) // 2
    g, r = grids(gpu, oracle, cfg, cap, sf.AuxMode.Variance)
    ref = reference_run(oracle, r, frames, intr, fusion, match, poses[0])
    assert ref[-1]["status"] == (5 if failure == "tracking_lost" else 4)
    die = len(ref) - 1
    assert die >= 2
    tr = sf.Tracker(g, intr, fusion, match, poses[0])
    for k, f in enumerate(frames):
        tr.step(f, sf.Tracker.TRACK)
        m = tr.fetch()
        if k < die:
            assert m.status == 0 and m.fusion == ref[k]["fusion"]
            assert pose_diff(m.pose, ref[k]["pose"]) < POSE_TOL
            continue
        assert m.status == ref[die]["status"]
        if k == die:
            assert m.registered == ref[die]["registered"]
            assert m.fusion == ref[die]["fusion"] == sf.FusionStats(0, 0, 0, 0)
            assert pose_diff(m.pose, ref[die]["pose"]) < POSE_TOL
            if not m.registered:
                assert m.iterations == 0 and m.matches == 0
            else:
                assert m.iterations == ref[die]["it"]
    assert_same_volume(g, r)


def test_reference_pose_chain_instability_and_fix(gpu):
    """The reference pose chain (pipeline.cpp:262-282) triples the rotation's departure from
    orthonormality every tracked frame; `orthonormalize` removes it."""
    intr = scenes.camera(160, 120, 131.25)
    poses = scenes.c1_trajectory(100)[:30]
    scene = scenes.sphere_plane_scene()
    frames = [gpu.render_synthetic_depth(scene, p, intr, domain_size=2.0) for p in poses]
    cfg = scenes.c1_config()
    fusion = sf.FusionParams(mode=sf.FusionMode.Weighted)
    match = sf.MatchParams.for_voxel_size(cfg.voxel_size)
    match.max_iterations = 0  # isolate the pose chain: delta = hook = exact ground-truth motion
    orth = {}
    for fix in (False, True):
        g = sf.SparseTsdfGrid(cfg, 0, sf.AuxMode.Weight)
        tr = sf.Tracker(g, intr, fusion, match, poses[0], orthonormalize=fix)
        errs = []
        for k, f in enumerate(frames):
            ext = sf.compose(sf.invert(poses[k - 1]), poses[k]) if k else sf.Pose.identity()
            tr.step(f, sf.Tracker.TRACK_WITH_HOOK, ext)
            R = tr.fetch().pose.rotation
            errs.append(np.abs(R.T @ R - np.eye(3)).max())
        orth[fix] = errs
    assert orth[False][25] > 1e4 * max(orth[False][3], 1e-16)  # exponential growth
    assert max(orth[True]) < 1e-14


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["fuse_kalman", "fuse_weighted_raycast", "icp"])
def test_golden_cases_gpu(gpu, name):
    """The CUDA path against the frozen reference outputs (tests/golden/golden.json, generated
    from the unmodified reference build): fusion, ray bounds, raycast and normals bit-exact;
    ICP pose within POSE_TOL (tree-ordered sums)."""
    import json
    import os

    from tests import golden_cases

    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden.json")) as f:
        want = json.load(f)["cases"][name]
    got = json.loads(json.dumps(golden_cases.CASES[name](gpu)))
    if name != "icp":
        assert got == want
        return
    d_got = np.array([float.fromhex(v) for v in got["delta"]])
    d_want = np.array([float.fromhex(v) for v in want["delta"]])
    assert np.abs(d_got - d_want).max() < POSE_TOL
    assert got["iterations"] == want["iterations"]
    assert abs(got["matches"] - want["matches"]) <= max(8, want["matches"] // 2000)
    assert got["gated"] == want["gated"]


@pytest.mark.parametrize("mode,steps", [(sf.FusionMode.Kalman, 2), (sf.FusionMode.Weighted, 4)])
def test_fuse_refinement_bit_exact(gpu, ref, mode, steps):
    """refinement_steps > 0 (fusion.cpp:99-143, bilinear depth + 0.5-px descent with libm's
    hypot) on noisy frames with a sigma plane: tables and payload codes equal the reference's."""
    intr = scenes.camera(160, 120, 131.25)
    poses = scenes.c1_trajectory(100)[::15][:4]
    frames = [gpu.render_synthetic_depth(scenes.sphere_plane_scene(), p, intr, sigma0=2.5e-4, seed=9 + k,
                                         domain_size=2.0) for k, p in enumerate(poses)]
    aux = sf.AuxMode.Variance if mode == sf.FusionMode.Kalman else sf.AuxMode.Weight
    g, r = grids(gpu, ref, scenes.c1_config(), 0, aux)
    params = sf.FusionParams(mode=mode, refinement_steps=steps)
    for f, p in zip(frames, poses):
        sg = gpu.fuse_frame(g, f, p, params)
        sr = ref.fuse_frame(r, f, p, params)
        assert sg == sr
        assert_same_volume(g, r)
    assert sr.voxels_updated > 1000


def test_tracker_streaming_fetch_matches_synchronous(gpu):
    """Host frames streamed (step k+1 issued before fetching step k; H2D overlaps compute)
    give the same per-frame metrics as step/fetch in lockstep, with or without the stage-timing
    events in the frame graph."""
    intr = scenes.camera(320, 240, 262.5)
    cfg = scenes.c1_config()
    poses = scenes.c1_trajectory(100)[:8]
    frames = [gpu.render_synthetic_depth(scenes.sphere_plane_scene(), p, intr, sigma0=2.5e-4, seed=21 + k,
                                         domain_size=2.0) for k, p in enumerate(poses)]
    fusion = sf.FusionParams(mode=sf.FusionMode.Kalman)
    match = sf.MatchParams.for_voxel_size(cfg.voxel_size)
    runs = []
    for streaming, level in ((False, 2), (True, 2), (False, 0)):
        grid = sf.SparseTsdfGrid(cfg, 0, sf.AuxMode.Variance)
        tr = sf.Tracker(grid, intr, fusion, match, poses[0])
        tr.set_stage_timing(level)  # stage events are graph nodes only: same results
        out = []
        for k, f in enumerate(frames):
            tr.step(f, sf.Tracker.TRACK)
            if not streaming:
                out.append(tr.fetch())
            elif k > 0:
                out.append(tr.fetch_frame(k - 1))
        if streaming:
            out.append(tr.fetch_frame(len(frames) - 1))
        st = tr.stage_times()
        assert (min(st) > 0) if level == 2 else (st == [-1.0] * 5)
        assert all(m.integrate_ns > 0 for m in out[1:])  # device-clock span of the integrate kernel
        runs.append([(m.frame, m.pose.to12().tobytes(), m.matches, m.fusion.voxels_updated, m.fusion.blocks_total,
                      m.raycast.hit_pixels) for m in out])
    assert runs[0] == runs[1] == runs[2]


def test_c3_room_fuse_and_raycast(gpu, oracle):
    """C3 (3 m room, 3000^3 at 1 mm: N = 375, not a power of two): Kalman fusion with a sigma
    plane, tables / payload codes / ray bounds / raycast equal the oracle's."""
    intr = scenes.camera(160, 120, 131.25)
    cfg = scenes.c3_config()
    poses = scenes.c3_trajectory(100)[::9][:3]
    frames = frames_for(gpu, scenes.c3_scene(), poses, intr, 3.0, sigma0=2.5e-4)
    g, r = grids(gpu, oracle, cfg, 400_000, sf.AuxMode.Variance)
    params = sf.FusionParams(mode=sf.FusionMode.Kalman)
    for f, p in zip(frames, poses):
        assert gpu.fuse_frame(g, f, p, params) == oracle.fuse_frame(r, f, p, params)
    assert_same_volume(g, r)
    assert r.allocated_count > 5000
    pose = poses[-1]
    tg, eg = gpu.compute_ray_bounds(g, pose, intr)
    tr, er = oracle.compute_ray_bounds(r, pose, intr)
    assert np.array_equal(tg.view(np.uint32), tr.view(np.uint32)) and np.array_equal(eg.view(np.uint32), er.view(np.uint32))
    dg, ng, sg = gpu.raycast_result(g, pose, intr)
    dr, nr, sr = oracle.raycast_result(r, pose, intr)
    assert np.array_equal(dg.depth.view(np.uint32), dr.depth.view(np.uint32))
    assert np.array_equal(ng.array.view(np.uint32), nr.array.view(np.uint32))
    assert (sg.sample_steps, sg.hit_pixels, sg.rays_with_bounds) == (sr.sample_steps, sr.hit_pixels, sr.rays_with_bounds)
    assert sg.hit_pixels > 500
