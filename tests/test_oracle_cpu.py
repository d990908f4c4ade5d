"""CPU suite: the C restatement (oracle/liboracle.so) pinned against the unmodified reference
build (oracle/_ref/libsfref.so) — bit-exact on every output — and against the reference's
own known-answer tests (proj/tests/test_grid.cpp, test_fusion.cpp, test_registration.cpp)."""
import math

import numpy as np
import pytest

from paper_1311_7194_b200 import api as sf
from tests import scenes


def pair(port, ref, cfg, cap, aux, **kw):
    return (sf.SparseTsdfGrid(cfg, cap, aux, backend=port, **kw), sf.SparseTsdfGrid(cfg, cap, aux, backend=ref, **kw))


def same_volume(a, b):
    assert np.array_equal(a.read_table(), b.read_table())
    assert np.array_equal(a.read_payload(), b.read_payload())
    assert a.allocated_count == b.allocated_count


# ---- reference known-answer tests, restated ---------------------------------------------
def test_quantizer_kats(port):
    """test_grid.cpp:25-40: 0 -> 0, delta -> 127, -delta -> -127, 1.5 delta -> 127 (clamped)."""
    cfg = sf.GridConfig(2, 4, (0, 0, 0), 1.0, 0.0)
    g = sf.SparseTsdfGrid(cfg, 8, backend=port)
    g.allocate_block([0, 0, 0])
    d = g.delta
    for t, code in [(0.0, 0), (d, 127), (-d, -127), (0.5 * d, 64)]:
        g.write_voxel([1, 1, 1], t, 1.0)
        raw = int(g.read_payload(0, 1)[(1 * 4 + 1) * 4 + 1]) & 0xFF
        assert np.int8(np.uint8(raw)) == code
    g.write_voxel([1, 1, 1], 1.5 * d, 1.0)  # |t| > delta is chi (grid.cpp:134)
    assert g.read_voxel([1, 1, 1]) is None


def test_roundtrip_within_half_code(port):
    """test_grid.cpp:42-51: round trip error <= delta/126."""
    cfg = sf.GridConfig(2, 4, (0, 0, 0), 1.0, 0.0)
    g = sf.SparseTsdfGrid(cfg, 8, backend=port)
    g.allocate_block([0, 0, 0])
    rng = np.random.default_rng(0)
    for t in rng.uniform(-g.delta, g.delta, 500):
        g.write_voxel([2, 1, 3], float(t), 1.0)
        assert abs(g.read_voxel([2, 1, 3])[0] - t) <= g.delta / 126.0


def test_slot_order_and_exhaustion(port):
    """test_grid.cpp:97-105: slot 0 first, idempotent, PoolExhausted."""
    cfg = sf.GridConfig(4, 4, (0, 0, 0), 1.0, 0.0)
    g = sf.SparseTsdfGrid(cfg, 2, backend=port)
    assert g.allocate_block([1, 2, 3]) == 0
    assert g.allocate_block([1, 2, 3]) == 0
    assert g.allocate_block([0, 0, 0]) == 1
    with pytest.raises(sf.PoolExhausted):
        g.allocate_block([3, 3, 3])
    g.free_block([1, 2, 3])
    assert g.allocate_block([2, 2, 2]) == 0  # LIFO free list (grid.cpp:106)
    assert g.memory_bytes() == 2 * 2 * 64 + 4 * 64


def test_measurement_kats(port, ref):
    """test_fusion.cpp:43-76: on-surface |T| < 1e-6, +-0.05 in front/behind, chi outside the band."""
    scene = sf.AnalyticScene()
    scene.add_plane([0.0, 0.0, -1.0], -2.0)
    intr = sf.Intrinsics.simple(64, 48, 55.0)
    frame = ref.render_synthetic_depth(scene, sf.Pose.identity(), intr)
    fp = sf.FusionParams(mode=sf.FusionMode.Simple, delta=0.1, edge_downweight=False, sigma0=2.5e-4)
    import ctypes as C
    from paper_1311_7194_b200 import _abi as A

    def meas(x):
        chi, t, var, w = C.c_int32(), C.c_double(), C.c_double(), C.c_double()
        fc, pc = frame.c(), fp.c()
        p12 = sf.Pose.identity().to12()
        xv = np.array(x, dtype=np.float64)
        assert ref.lib.estimate_measurement(C.byref(fc), p12.ctypes.data_as(A.c_double_p),
                                            xv.ctypes.data_as(A.c_double_p), C.byref(pc), C.byref(chi),
                                            C.byref(t), C.byref(var), C.byref(w)) == 0
        return None if chi.value else (t.value, var.value, w.value)

    on = meas([0.0, 0.0, 2.0])
    assert abs(on[0]) < 1e-6 and abs(on[1] - 1e-6) < 1e-9 and on[2] == 0.1
    assert abs(meas([0.0, 0.0, 1.95])[0] - 0.05) < 1e-4
    assert abs(meas([0.0, 0.0, 2.05])[0] + 0.05) < 1e-4
    for x in ([0, 0, 1.8], [0, 0, 2.2], [0, 0, -1.0], [5.0, 0, 2.0]):
        assert meas(x) is None


# ---- bit-exact restatement vs the reference build -----------------------------------------
def small_cam():
    return scenes.camera(160, 120, 131.25)


@pytest.mark.parametrize("mode", [sf.FusionMode.Kalman, sf.FusionMode.Weighted, sf.FusionMode.Simple])
def test_fuse_frame_bit_exact(port, ref, mode):
    intr = small_cam()
    poses = scenes.c1_trajectory(100)[::30]
    aux = sf.AuxMode.Variance if mode == sf.FusionMode.Kalman else sf.AuxMode.Weight
    a, b = pair(port, ref, scenes.c1_config(), 0, aux)
    params = sf.FusionParams(mode=mode)
    for p in poses:
        f = ref.render_synthetic_depth(scenes.sphere_plane_scene(), p, intr, sigma0=2.5e-4, seed=5, domain_size=2.0)
        assert port.fuse_frame(a, f, p, params) == ref.fuse_frame(b, f, p, params)
        same_volume(a, b)


def test_refinement_path_bit_exact(port, ref):
    """fusion.cpp:99-143 (refinement_steps > 0), restated in the oracle."""
    intr = small_cam()
    p = scenes.c1_trajectory(100)[20]
    a, b = pair(port, ref, scenes.c1_config(), 0, sf.AuxMode.Weight)
    params = sf.FusionParams(mode=sf.FusionMode.Weighted, refinement_steps=3)
    f = ref.render_synthetic_depth(scenes.sphere_plane_scene(), p, intr, domain_size=2.0)
    assert port.fuse_frame(a, f, p, params) == ref.fuse_frame(b, f, p, params)
    same_volume(a, b)


def test_pool_exhaustion_prefix(port, ref):
    intr = small_cam()
    p = scenes.c1_trajectory(100)[10]
    a, b = pair(port, ref, scenes.c1_config(), 60, sf.AuxMode.Weight)
    f = ref.render_synthetic_depth(scenes.sphere_plane_scene(), p, intr, domain_size=2.0)
    with pytest.raises(sf.PoolExhausted):
        ref.fuse_frame(b, f, p, sf.FusionParams())
    with pytest.raises(sf.PoolExhausted):
        port.fuse_frame(a, f, p, sf.FusionParams())
    same_volume(a, b)


def test_lists_bounds_raycast_normals_bit_exact(port, ref):
    intr = small_cam()
    poses = scenes.c1_trajectory(100)
    scene = scenes.sphere_plane_scene()
    a, b = pair(port, ref, scenes.c1_config(), 0, sf.AuxMode.Weight)
    for p in poses[:60:20]:
        f = ref.render_synthetic_depth(scene, p, intr, domain_size=2.0)
        la, lb = port.select_update_blocks(a, f, p), ref.select_update_blocks(b, f, p)
        assert np.array_equal(la[0], lb[0]) and np.array_equal(la[1], lb[1])
        port.fuse_frame(a, f, p, sf.FusionParams(mode=sf.FusionMode.Weighted))
        ref.fuse_frame(b, f, p, sf.FusionParams(mode=sf.FusionMode.Weighted))
    same_volume(a, b)
    q = poses[30]
    sa, ea = port.compute_ray_bounds(a, q, intr)
    sb, eb = ref.compute_ray_bounds(b, q, intr)
    assert np.array_equal(sa, sb) and np.array_equal(ea, eb)
    da, na, sta = port.raycast_result(a, q, intr)
    db, nb, stb = ref.raycast_result(b, q, intr)
    assert sta == stb and sta.hit_pixels > 1000
    assert np.array_equal(da.depth, db.depth) and np.array_equal(na.array, nb.array)
    f = ref.render_synthetic_depth(scene, q, intr, sigma0=2.5e-4, seed=9, domain_size=2.0)
    assert np.array_equal(port.compute_normals(f, 2.5e-4, 0.0078).array, ref.compute_normals(f, 2.5e-4, 0.0078).array)


def test_icp_bit_exact(port, ref):
    """The sequential Kahan sums of the restatement reproduce the reference pose bit for bit."""
    intr = small_cam()
    scene = scenes.cluster_scene()
    tp = sf.orbit_trajectory([0.0, 0.0, 1.3], 1.3, 8)[1]
    ang = math.radians(2.0)
    sp = sf.compose(tp, sf.Pose([[math.cos(ang), 0, math.sin(ang)], [0, 1, 0], [-math.sin(ang), 0, math.cos(ang)]],
                                [0.01, -0.005, 0.008]))
    t = ref.render_synthetic_depth(scene, tp, intr)
    s = ref.render_synthetic_depth(scene, sp, intr)
    tn = ref.compute_normals(t, 2.5e-4, 0.006)
    params = sf.MatchParams.for_voxel_size(1.5 / 256.0)
    ra = port.icp(s, t, tn, sf.Pose.identity(), params)
    rb = ref.icp(s, t, tn, sf.Pose.identity(), params)
    assert np.array_equal(ra.delta.to12(), rb.delta.to12())
    assert ra.iterations == rb.iterations and ra.matches == rb.matches
    assert ra.eigenvalues == rb.eigenvalues and ra.gated_mask == rb.gated_mask


def test_synthetic_depth_bit_exact(port, ref):
    intr = small_cam()
    scene = scenes.sphere_plane_scene()
    scene.add_box([0.3, -0.2, 1.0], [0.1, 0.05, 0.08])
    p = scenes.c1_trajectory(10)[3]
    a = port.render_synthetic_depth(scene, p, intr, domain_size=2.0)
    b = ref.render_synthetic_depth(scene, p, intr, domain_size=2.0)
    assert np.array_equal(a.depth, b.depth)


def test_tracking_lost(port, ref):
    intr = sf.Intrinsics.simple(32, 24, 28.0)
    z = sf.DepthFrame(intr, np.zeros((24, 32), np.float32))
    n = sf.NormalMap(np.zeros((24, 32, 3), np.float32))
    for be in (port, ref):
        with pytest.raises(sf.TrackingLost):
            be.icp(z, z, n, sf.Pose.identity(), sf.MatchParams())


def test_invalid_arguments_mirror_reference(port, ref):
    for be in (port, ref):
        with pytest.raises(ValueError):
            sf.SparseTsdfGrid(sf.GridConfig(0, 8, (0, 0, 0), 1.0, 0.0), backend=be)
        with pytest.raises(ValueError):
            sf.SparseTsdfGrid(sf.GridConfig(4, 4, (0, 0, 0), 1.0, 0.0), 65, backend=be)
        g = sf.SparseTsdfGrid(sf.GridConfig(4, 4, (0, 0, 0), 1.0, 0.0), 8, backend=be)
        with pytest.raises(IndexError):
            g.allocate_block([4, 0, 0])
        with pytest.raises(RuntimeError):
            g.write_voxel([0, 0, 0], 0.0, 1.0)
        intr = small_cam()
        f = sf.DepthFrame(intr, np.zeros((120, 160), np.float32))
        with pytest.raises(ValueError):  # Kalman on a weight-mode grid (fusion.cpp:279-283)
            be.fuse_frame(g, f, sf.Pose.identity(), sf.FusionParams(mode=sf.FusionMode.Kalman))
        with pytest.raises(ValueError):
            be.fuse_frame(g, f, sf.Pose.identity(), sf.FusionParams(w_fixed=1.5))


def test_glibc_hypot_is_the_restated_kernel():
    """The device refinement path (csrc/sf_fusion.cu glibc_hypot) restates the reference libm's
    hypot: the non-FMA Borges kernel. Pin: identical to libm.hypot on random pairs across the
    magnitudes of the refinement gradients (it is not correctly rounded, so the sequence matters)."""
    import ctypes
    import math
    import random

    libm = ctypes.CDLL("libm.so.6")
    libm.hypot.restype = ctypes.c_double
    libm.hypot.argtypes = [ctypes.c_double, ctypes.c_double]

    def kernel(ax, ay):
        h = math.sqrt(ax * ax + ay * ay)
        if h <= 2.0 * ay:
            d = h - ay
            t1 = ax * (2.0 * d - ax)
            t2 = (d - 2.0 * (ax - ay)) * d
        else:
            d = h - ax
            t1 = 2.0 * d * (ax - 2.0 * ay)
            t2 = (4.0 * d - ay) * ay + d * d
        return h - (t1 + t2) / (2.0 * h)

    def hyp(x, y):
        x, y = abs(x), abs(y)
        ax, ay = (y, x) if x < y else (x, y)
        if ay <= ax * 2.0 ** -54:
            return ax + ay
        return kernel(ax, ay)

    rng = random.Random(7)
    for _ in range(20000):
        a = rng.uniform(-1, 1) * 10 ** rng.uniform(-9, 1)
        b = rng.uniform(-1, 1) * 10 ** rng.uniform(-9, 1)
        assert hyp(a, b) == libm.hypot(a, b), (a, b)
