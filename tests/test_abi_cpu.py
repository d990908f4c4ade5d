"""CPU-only checks: the C-ABI library loads and exports every declared entry point, the
host-side codec tables and pose math are exact against the reference (no GPU calls)."""
import ctypes as C
import math
import os
import re

import numpy as np
import pytest

from paper_1311_7194_b200 import _abi as A
from paper_1311_7194_b200 import api as sf
from tests import scenes

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "sf_gpu.h")).read()
    return sorted(set(re.findall(r"^(?:int|int32_t|const char\*)\s+(sf_[a-z0-9_]+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(A.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # and the ctypes mirror covers them all
    assert set(A.EXPORTED) <= set(syms) | {"sf_version"}


def test_version_string():
    assert A.product().version().decode().startswith("sf_gpu")


def test_native_library_is_sm100a_only():
    out = os.popen(f"cuobjdump --list-elf {A.LIB_PATH} 2>/dev/null").read()
    if not out:
        pytest.skip("cuobjdump unavailable")
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def _lround(x):
    # std::lround on a finite double (half away from zero), exact
    r = math.floor(abs(x))
    frac = abs(x) - r
    v = r + (1 if frac >= 0.5 else 0)
    return int(math.copysign(v, x)) if x != 0 else 0


def _ref_encode_variance(v, p_min, p_max):
    # AuxQuantization::encode, variance branch (grid.cpp:43-45)
    c = min(max(v, p_min), p_max)
    s = math.log(c / p_min) / math.log(p_max / p_min)
    return _lround(s * 255.0) & 0xFF


@pytest.mark.parametrize("p_min,p_max", [(1e-8, 1e-2), (1e-12, 1e-2), (1e-10, 1e-4)])
def test_variance_threshold_encode_matches_log_encode(p_min, p_max):
    lib = A.product()
    aux = A.AuxQuantC(1, 20.0, p_min, p_max)
    td = (C.c_double * 256)()
    ad = (C.c_double * 256)()
    th = (C.c_double * 256)()
    assert lib.debug_aux_tables(C.byref(aux), 0.01, td, ad, th) == 0
    thr = np.array(list(th))
    assert np.all(np.diff(thr[1:]) > 0)
    rng = np.random.default_rng(1)
    vals = np.exp(rng.uniform(math.log(p_min) - 2, math.log(p_max) + 2, 20000))
    # plus the thresholds themselves and their neighbours (the only places a code flips)
    edge = np.concatenate([thr[1:], np.nextafter(thr[1:], 0), np.nextafter(thr[1:], 1)])
    for v in np.concatenate([vals, edge]):
        code = int(np.searchsorted(thr[1:], v, side="right"))
        assert code == _ref_encode_variance(float(v), p_min, p_max), v


def test_variance_codes_against_reference_write_voxel(ref):
    """The threshold encode reproduces the reference's own encode through its public API."""
    p_min, p_max = 1e-12, 1e-2
    lib = A.product()
    aux = A.AuxQuantC(1, 20.0, p_min, p_max)
    td, ad, th = (C.c_double * 256)(), (C.c_double * 256)(), (C.c_double * 256)()
    lib.debug_aux_tables(C.byref(aux), 0.01, td, ad, th)
    thr = np.array(list(th))
    cfg = sf.GridConfig(2, 8, (0, 0, 0), 1.0, 0.0)
    g = sf.SparseTsdfGrid(cfg, 8, sf.AuxMode.Variance, p_min=p_min, p_max=p_max, backend=ref)
    g.allocate_block([0, 0, 0])
    rng = np.random.default_rng(7)
    vals = np.concatenate([np.exp(rng.uniform(math.log(p_min) - 1, math.log(p_max) + 1, 400)),
                           thr[1:], np.nextafter(thr[1:], 0)])
    for i, v in enumerate(vals):
        g.write_voxel([i % 8, (i // 8) % 8, 0], 0.0, float(v))
        code = int(g.read_payload(0, 1)[(i // 8 % 8) * 8 + i % 8]) >> 8
        assert code == int(np.searchsorted(thr[1:], v, side="right")), v
        # decode table == reference decode
        assert g.read_voxel([i % 8, (i // 8) % 8, 0])[1] == ad[code]


def test_pose_math_bit_exact(ref):
    rng = np.random.default_rng(3)
    lib = ref.lib
    for _ in range(50):
        q = rng.normal(size=4)
        q /= np.linalg.norm(q)
        w, x, y, z = q
        R = np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                      [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                      [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])
        a = sf.Pose(R, rng.normal(size=3))
        b = sf.Pose(R.T, rng.normal(size=3))
        out = (C.c_double * 12)()
        a12, b12 = a.to12(), b.to12()
        lib.compose(a12.ctypes.data_as(A.c_double_p), b12.ctypes.data_as(A.c_double_p), out)
        assert np.array_equal(sf.compose(a, b).to12(), np.array(list(out)))
        lib.invert(a12.ctypes.data_as(A.c_double_p), out)
        assert np.array_equal(sf.invert(a).to12(), np.array(list(out)))


@pytest.mark.parametrize("frames,arc", [(100, math.pi / 2), (8, 2 * math.pi), (1, 1.0)])
def test_orbit_trajectory_bit_exact(ref, frames, arc):
    poses = sf.orbit_trajectory([0.0, 0.0, 1.3], 1.3, frames, (0.0, 1.0, 0.0), math.pi / 4, arc)
    out = np.zeros(12 * frames)
    tgt = np.array([0.0, 0.0, 1.3])
    ax = np.array([0.0, 1.0, 0.0])
    ref.lib.orbit_trajectory(tgt.ctypes.data_as(A.c_double_p), 1.3, frames, ax.ctypes.data_as(A.c_double_p),
                             math.pi / 4, arc, out.ctypes.data_as(A.c_double_p))
    for k, p in enumerate(poses):
        assert np.array_equal(p.to12(), out[12 * k: 12 * k + 12])


def test_reference_wrapper_fuses_on_cpu(ref):
    intr = scenes.camera(160, 120, 131.25)
    scene = scenes.sphere_plane_scene()
    pose = scenes.c1_trajectory(4)[0]
    frame = ref.render_synthetic_depth(scene, pose, intr, domain_size=2.0)
    g = sf.SparseTsdfGrid(scenes.c1_config(), 0, sf.AuxMode.Variance, backend=ref)
    st = ref.fuse_frame(g, frame, pose, sf.FusionParams(mode=sf.FusionMode.Kalman))
    assert st.blocks_total > 20 and st.voxels_updated > 1000
    assert st.memory_bytes == 2 * st.blocks_total * 512 + 4 * 32 ** 3
    assert ref.lib.volume_check_consistency(g.handle) == 0


def test_dfrm_files_match_reference(tmp_path):
    """DFRM write is byte-identical to the reference's write_dfrm; read applies its
    out-of-range rule (frame_io.cpp:28-79). Host buffers only: no GPU needed."""
    from tests import oracle_backends

    ref = oracle_backends.reference()
    if ref is None:
        pytest.skip("reference build absent")
    gpu = sf.default_backend()
    intr = sf.Intrinsics.simple(40, 30, 35.0, 0.2, 3.0)
    rng = np.random.default_rng(5)
    depth = rng.uniform(0.0, 4.0, (30, 40)).astype(np.float32)
    depth[::7, ::5] = 0.0
    sigma = rng.uniform(0.0, 0.01, (30, 40)).astype(np.float32)
    for sg in (None, sigma):
        f = sf.DepthFrame(intr, depth, sg)
        a, b = str(tmp_path / "a.dfrm"), str(tmp_path / "b.dfrm")
        gpu.write_dfrm(f, a)
        ref.write_dfrm(f, b)
        assert open(a, "rb").read() == open(b, "rb").read()
        ra, rb = gpu.read_dfrm(a), ref.read_dfrm(b)
        assert np.array_equal(ra.depth.view(np.uint32), rb.depth.view(np.uint32))
        assert (ra.sigma is None) == (sg is None) == (rb.sigma is None)
        if sg is not None:
            assert np.array_equal(ra.sigma, rb.sigma)
        assert (ra.intrinsics.width, ra.intrinsics.height) == (40, 30)
        assert np.all((ra.depth == 0) | ((ra.depth >= np.float32(0.2)) & (ra.depth <= np.float32(3.0))))


def test_trajectory_csv_matches_reference(tmp_path):
    """Trajectory CSV (frame_io.cpp:81-126): write byte-identical to write_trajectory; read
    equal bit for bit, incl. 12-value rows, '#' comments, empty lines and the nearest-rotation
    repair of a non-orthonormal row. Host-side I/O: no GPU needed."""
    from tests import oracle_backends

    ref = oracle_backends.reference()
    if ref is None:
        pytest.skip("reference build absent")
    gpu = sf.default_backend()
    poses = sf.orbit_trajectory([0.1, -0.2, 1.3], 1.3, 7, (0.0, 1.0, 0.0), 0.3, 1.1)
    entries = [(3 * k + 1, p) for k, p in enumerate(poses)]
    a, b = str(tmp_path / "a.csv"), str(tmp_path / "b.csv")
    gpu.write_trajectory(entries, a)
    ref.write_trajectory(entries, b)
    assert open(a, "rb").read() == open(b, "rb").read()
    # hand-written rows: a comment, a blank line, a 12-value row, a slightly skewed rotation
    skew = "0,1.0,1e-4,0,0,1,0,0,0,1,0.5,0.25,2"
    text = "# frame,r00..r22,t\n\n" + open(a).read() + "1,0,0,0,1,0,0,0,1,-1,0,3\n" + skew + "\n"
    c = tmp_path / "c.csv"
    c.write_text(text)
    ra, rb = gpu.read_trajectory(str(c)), ref.read_trajectory(str(c))
    assert len(ra) == len(rb) == len(entries) + 2
    for (fa, pa), (fb, pb) in zip(ra, rb):
        assert fa == fb
        assert np.array_equal(pa.to12(), pb.to12())
    assert ra[-2][0] == 0 and ra[-1][1].rotation[0, 1] != 1e-4  # repaired by nearest_rotation
    bad = tmp_path / "bad.csv"
    bad.write_text("1,2,3\n")
    with pytest.raises(RuntimeError):
        gpu.read_trajectory(str(bad))
